"""Random 1-byte gather over 333 MB with different load flavours (DRAM fetch size study).

  python tools/gather_modes.py            # timing of every mode
  python tools/gather_modes.py --one M    # a single launch of mode M (for ncu)
"""
import argparse
import ctypes as C
import json
import os

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
bench = C.CDLL(os.path.join(ROOT, "paper_2502_15539_b200", "libph_bench.so"))
bench.phb_gather_mode.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int,
                                  C.c_void_p, C.c_void_p]
NAMES = ["nc.L1::no_allocate.L2::cache_hint(evict_last)", "nc", "cg", "cv", "nc.L2::64B",
         "nc.L2::128B", "nc.L2::256B", "lu", "cs", "plain"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--one", type=int, default=-1)
    ap.add_argument("--mb", type=int, default=333)
    a = ap.parse_args()
    s = torch.cuda.current_stream()
    sp = C.c_void_p(s.cuda_stream)
    F = a.mb << 20
    buf = torch.ones(F, dtype=torch.uint8, device="cuda")
    sink = torch.zeros(1, dtype=torch.int32, device="cuda")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    nl = 1 << 28
    if a.one >= 0:
        bench.phb_gather_mode(buf.data_ptr(), F, nl, 9, a.one, sink.data_ptr(), sp)
        torch.cuda.synchronize()
        return
    for m, name in enumerate(NAMES):
        bench.phb_gather_mode(buf.data_ptr(), F, nl, 9, m, sink.data_ptr(), sp)
        best = 1e9
        for _ in range(3):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            bench.phb_gather_mode(buf.data_ptr(), F, nl, 9, m, sink.data_ptr(), sp)
            e1.record(s)
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
        print(json.dumps({"mode": m, "load": name, "mb": a.mb,
                          "gloads_s": round(nl / best / 1e6, 2)}), flush=True)


if __name__ == "__main__":
    main()
