"""L1->XBAR request-port model of pass B (not the product): the L2-resident random 1-byte
gather rate over a 32 MiB buffer, alone and with coalesced streams beside it (8 or 16 B in,
4 or 8 B out per gather), in pass B's launch shape (4 x 256 threads per SM, 8 gathers per
thread in flight). If the port takes one 32-B sector per cycle per SM whatever the sector's
origin, the time per gather grows by (streamed bytes / 32) port slots:

    t(in, out) ~= t(0, 0) * (1 + in/32 + out/32)

  python tools/port_model.py [--mb 32] [--n 500000000] [--out profiles/r02_port_model.jsonl]
"""
import argparse
import ctypes as C
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mb", type=int, default=32)
    ap.add_argument("--n", type=int, default=500_000_000)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    lib = C.CDLL(os.path.join(ROOT, "paper_2502_15539_b200", "libph_bench.so"))
    lib.phb_port_model.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, C.c_int,
                                   C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    F = a.mb << 20
    n = a.n // 256 * 256
    buf = torch.randint(0, 255, (F,), dtype=torch.uint8, device="cuda")
    sin = torch.randint(-2**62, 2**62, (2 * n,), dtype=torch.int64, device="cuda")
    sout = torch.empty(n, dtype=torch.int64, device="cuda")
    sink = torch.zeros(1, dtype=torch.int32, device="cuda")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    clk = torch.cuda.clock_rate() * 1e6 if hasattr(torch.cuda, "clock_rate") else 1.965e9
    st = torch.cuda.current_stream().cuda_stream
    rows = []
    base = None
    for in_w, out_b in ((0, 0), (1, 0), (2, 0), (0, 4), (1, 4), (1, 42), (1, 44), (1, -4), (1, 8), (2, 4), (2, 8)):  # -4: bulk stores
        def run():
            assert lib.phb_port_model(buf.data_ptr(), F, n, 7, in_w, out_b, sin.data_ptr(),
                                      sout.data_ptr(), sink.data_ptr(), st) == 0
        run()
        run()
        torch.cuda.synchronize()
        ts = []
        for _ in range(a.reps):
            flush.fill_(1)
            run()  # warm the 32 MiB buffer into L2 again after the flush
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            run()
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = min(ts)
        if base is None:
            base = ms
        ob = 4 if out_b in (42, 44) else abs(out_b)
        sect = 1 + in_w * 8 / 32 + ob / 32
        row = {"buffer_mb": a.mb, "gathers": n, "in_bytes": in_w * 8, "out_bytes": ob, "out_path": ("smem + cp.async.bulk" if out_b < 0 else "st.global.cs.v2.u32" if out_b == 42
                                                 else "st.global.cs.v4.u32" if out_b == 44 else "st.global.cs"),
               "ms": round(ms, 4), "ggathers_s": round(n / ms / 1e6, 2),
               "port_sectors_per_gather": round(sect, 4),
               "gsectors_s": round(n * sect / ms / 1e6, 2),
               "sectors_per_clk_per_sm": round(n * sect / (ms * 1e-3) / (sms * clk), 4),
               "t_over_t00": round(ms / base, 4), "model_t_over_t00": round(sect, 4)}
        rows.append(row)
        print(json.dumps(row), flush=True)
    if a.out:
        with open(a.out, "w") as f:
            for r in rows:
                f.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
