"""PCIe bounds for the e2e path: pinned H2D and D2H bandwidth alone and overlapped
(the ceiling for ph_gpu_index_stream_* at 8 B in + 4 B out per key)."""
import json
import time

import torch


def main():
    n = 8 << 30
    h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
    h_out = torch.empty(n // 2, dtype=torch.uint8).pin_memory()
    d_in = torch.empty(n, dtype=torch.uint8, device="cuda")
    d_out = torch.empty(n // 2, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    res = {}
    for name, fn in (("h2d_8GB", lambda: d_in.copy_(h_in, non_blocking=True)),
                     ("d2h_4GB", lambda: h_out.copy_(d_out, non_blocking=True))):
        fn()
        torch.cuda.synchronize()
        t = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        res[name + "_GBps"] = round((n if name.startswith("h2d") else n // 2) / dt / 1e9, 2)
    torch.cuda.synchronize()
    t = time.perf_counter()
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    res["overlapped_8GB_in_4GB_out_ms"] = round(dt * 1e3, 1)
    res["e2e_bound_gkeys_s_at_12B"] = round(1e9 / dt / 1e9 * (n / 8) / 1e9, 3)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
