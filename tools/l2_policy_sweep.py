"""Does any L2 mechanism keep a hot subset resident under a random gather? (characterisation)

Skewed gather over a 333 MB buffer: p_hot of the loads go to the first F_hot bytes.
Compares: hints off, evict_last everywhere, hot evict_last + cold evict_first, and a
persisting access-policy window over the hot region (with each hint mode).
"""
import ctypes as C
import json
import os

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
bench = C.CDLL(os.path.join(ROOT, "paper_2502_15539_b200", "libph_bench.so"))
bench.phb_gather_skew.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_double, C.c_uint64,
                                  C.c_uint64, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                  C.c_void_p]
bench.phb_set_persist.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_float, C.c_size_t]
bench.phb_max_persist_bytes.restype = C.c_longlong


def main():
    s = torch.cuda.current_stream()
    sp = C.c_void_p(s.cuda_stream)
    F = 333 << 20
    buf = torch.ones(F, dtype=torch.uint8, device="cuda")
    sink = torch.zeros(1, dtype=torch.int32, device="cuda")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    nl = 1 << 28
    maxp = bench.phb_max_persist_bytes()

    sin = torch.empty(nl, dtype=torch.int64, device="cuda")
    sout = torch.empty(nl, dtype=torch.int32, device="cuda")
    streaming = [False]

    def t(F_hot, p_hot, mode):
        def run():
            bench.phb_gather_skew(buf.data_ptr(), F_hot, F, p_hot, nl, 5, mode, sink.data_ptr(), sp,
                                  sin.data_ptr() if streaming[0] else None,
                                  sout.data_ptr() if streaming[0] else None)
        run()
        best = 1e9
        for _ in range(3):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            run()
            b.record(s)
            b.synchronize()
            best = min(best, a.elapsed_time(b))
        return round(nl / best / 1e6, 2)

    for (hot_mb, p_hot), stream_on in [(hp, so) for so in (False, True)
                                       for hp in ((32, 0.37), (48, 0.45), (64, 0.5), (96, 0.6))]:
        streaming[0] = stream_on
        Fh = hot_mb << 20
        r = {"hot_mb": hot_mb, "p_hot": p_hot, "with_12B_stream": stream_on}
        for mode, name in ((2, "nohint"), (0, "all_last"), (1, "hot_last_cold_first")):
            r[name] = t(Fh, p_hot, mode)
        for carve_mb in (int(maxp) >> 20,):
            bench.phb_set_persist(sp, buf.data_ptr(), min(Fh, maxp), 1.0, maxp)
            for mode, name in ((2, "persist_nohint"), (1, "persist_hot_last_cold_first")):
                r[name] = t(Fh, p_hot, mode)
            bench.phb_set_persist(sp, buf.data_ptr(), 0, 0.0, 0)
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
