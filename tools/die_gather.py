"""Does die-local access double the effective L2 for a random gather? (characterisation)

Probes every 2 KiB chunk of a 512 MiB buffer from one thread on every SM (ld.global.cv
latency), derives each SM's die (agreement of its near/far split with SM 0's) and each
chunk's home die (mean latency from die-0 SMs minus die-1 SMs), then times random 1-byte
gathers where SMs read only chunks homed on their own die (mode 0) versus the same chunk
sets read by every SM (mode 1), at several footprints.
"""
import ctypes as C
import json
import os

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
bench = C.CDLL(os.path.join(ROOT, "paper_2502_15539_b200", "libph_bench.so"))
bench.phb_die_probe.argtypes = [C.c_void_p, C.c_uint64, C.c_uint32, C.c_int, C.c_void_p,
                                C.c_void_p, C.c_int, C.c_void_p]
bench.phb_gather_die.argtypes = [C.c_void_p, C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint32,
                                 C.c_void_p, C.c_uint32, C.c_uint64, C.c_uint64, C.c_int,
                                 C.c_void_p, C.c_void_p]


def main():
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--only-mb", type=int, default=0, help="one footprint, one run per mode (ncu)")
    args = ap.parse_args()
    s = torch.cuda.current_stream()
    sp = C.c_void_p(s.cuda_stream)
    chunk = 2048
    nchunks = (512 << 20) // chunk
    buf = torch.ones(nchunks * chunk // 4, dtype=torch.int32, device="cuda")
    blocks = 148
    lat = torch.zeros(blocks * nchunks, dtype=torch.int32, device="cuda")
    smid = torch.zeros(blocks, dtype=torch.int32, device="cuda")
    bench.phb_die_probe(buf.data_ptr(), nchunks, chunk, blocks, lat.data_ptr(), smid.data_ptr(),
                        2, sp)
    torch.cuda.synchronize()
    L = lat.cpu().numpy().reshape(blocks, nchunks).astype(np.float64)
    sm = smid.cpu().numpy()
    med = np.median(L, axis=1, keepdims=True)
    cls = L > med
    agree = (cls == cls[0]).mean(axis=1)
    die_of_block = (agree < 0.5).astype(np.int8)
    sm_die = np.zeros(256, dtype=np.int8)
    for b in range(blocks):
        sm_die[sm[b]] = die_of_block[b]
    d0 = L[die_of_block == 0].mean(axis=0)
    d1 = L[die_of_block == 1].mean(axis=0)
    home = (d0 > d1).astype(np.int8)  # home die = the die with the lower latency
    margin = np.abs(d0 - d1)
    print(json.dumps({"sms_die0": int((die_of_block == 0).sum()), "sms_die1": int((die_of_block == 1).sum()),
                      "chunks_home0": int((home == 0).sum()), "chunks_home1": int((home == 1).sum()),
                      "latency_margin_p5_p50": [float(np.percentile(margin, 5)), float(np.median(margin))]}),
          flush=True)
    if (home == 0).sum() == 0 or (home == 1).sum() == 0 or (die_of_block == 1).sum() == 0:
        print(json.dumps({"error": "no die split found"}))
        return
    l0 = torch.from_numpy(np.nonzero(home == 0)[0].astype(np.int32)).cuda()
    l1 = torch.from_numpy(np.nonzero(home == 1)[0].astype(np.int32)).cuda()
    smd = torch.from_numpy(sm_die).cuda()
    sink = torch.zeros(1, dtype=torch.int32, device="cuda")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    nl = 1 << 28
    for mb in ((args.only_mb,) if args.only_mb else (32, 64, 96, 128, 160, 192, 256, 333)):
        per = (mb << 20) // 2 // chunk
        n0, n1 = min(per, l0.numel()), min(per, l1.numel())
        r = {"footprint_mb": mb}
        for mode, name in ((0, "die_local"), (1, "mixed")):
            def run():
                bench.phb_gather_die(buf.data_ptr(), l0.data_ptr(), n0, l1.data_ptr(), n1,
                                     smd.data_ptr(), chunk, nl, 7, mode, sink.data_ptr(), sp)
            run()
            if args.only_mb:
                continue
            best = 1e9
            for _ in range(3):
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(s)
                run()
                b.record(s)
                b.synchronize()
                best = min(best, a.elapsed_time(b))
            r[name + "_gloads_s"] = round(nl / best / 1e6, 2)
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
