"""Random-gather microbenchmark sweep (roofline characterisation, not the product).

For buffers of F bytes, times 2^28 uniformly random 1-byte loads (the query kernel's load
instruction and L2 policy) and reports G sectors/s; then the same with the L2 fetch
granularity limit at 32 B. Optionally --ncu runs a single gather at --ncu-mb.
"""
import argparse
import ctypes as C
import json
import os

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
bench = C.CDLL(os.path.join(ROOT, "paper_2502_15539_b200", "libph_bench.so"))
bench.phb_get_l2_fetch_granularity.restype = C.c_longlong


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ncu", action="store_true")
    ap.add_argument("--ncu-mb", type=int, default=333)
    args = ap.parse_args()
    s = torch.cuda.current_stream()
    sp = C.c_void_p(s.cuda_stream)
    sink = torch.zeros(1, dtype=torch.int32, device="cuda")
    nl = 1 << 28
    big = torch.ones(2 << 30, dtype=torch.uint8, device="cuda")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")

    def run(F, kpt=8, bps=8):
        bench.phb_gather(C.c_void_p(big.data_ptr()), C.c_uint64(F), C.c_uint64(nl), C.c_uint64(3),
                         kpt, bps, C.c_void_p(sink.data_ptr()), sp)

    if args.ncu:
        run(args.ncu_mb << 20)
        torch.cuda.synchronize()
        return

    def t(F, **kw):
        run(F, **kw)
        best = 1e9
        for _ in range(3):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            run(F, **kw)
            b.record(s)
            b.synchronize()
            best = min(best, a.elapsed_time(b))
        return nl / best / 1e6

    g0 = bench.phb_get_l2_fetch_granularity()
    for gran in (g0, 32):
        bench.phb_set_l2_fetch_granularity(gran)
        for mb in (4, 16, 32, 48, 64, 80, 96, 128, 192, 256, 333, 512, 1024, 2048):
            print(json.dumps({"fetch": gran, "mb": mb, "gsectors_s": round(t(mb << 20), 2)}),
                  flush=True)
    bench.phb_set_l2_fetch_granularity(g0)
    for kpt in (1, 4, 8, 16):
        for bps in (2, 4, 8):
            print(json.dumps({"mb": 333, "kpt": kpt, "bps": bps,
                              "gsectors_s": round(t(333 << 20, kpt=kpt, bps=bps), 2)}), flush=True)


if __name__ == "__main__":
    main()
