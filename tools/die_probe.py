"""Dual-die L2 probe (characterisation, not the product).

1. One thread on one SM times ld.global.cv to the first word of every 2 KiB chunk of a
   buffer: the latency histogram shows whether chunks are homed on the near or far die.
2. The same chunks probed from a thread on several other SMs: do SMs agree on the split
   (classification consistent up to a global flip per die)?
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


def main():
    s = torch.cuda.current_stream()
    sp = C.c_void_p(s.cuda_stream)
    chunk = 2048
    nchunks = 4096  # 8 MiB
    buf = torch.ones(nchunks * chunk // 4, dtype=torch.int32, device="cuda")
    blocks = 148 * 2
    lat = torch.zeros(blocks * nchunks, dtype=torch.int32, device="cuda")
    smid = torch.zeros(blocks, dtype=torch.int32, device="cuda")
    bench.phb_die_probe(buf.data_ptr(), nchunks, chunk, blocks, lat.data_ptr(), smid.data_ptr(), 2, sp)
    torch.cuda.synchronize()
    L = lat.cpu().numpy().reshape(blocks, nchunks)
    sm = smid.cpu().numpy()
    h = np.bincount(np.clip(L[0], 0, 2000) // 10)
    top = sorted(((int(c), int(b * 10)) for b, c in enumerate(h) if c), reverse=True)[:8]
    print(json.dumps({"sm": int(sm[0]), "latency_hist_top(count, cycles)": top,
                      "median": float(np.median(L[0]))}))
    thr = np.median(L[0])
    cls0 = L[0] > thr
    agree = []
    for b in range(1, blocks):
        c = L[b] > np.median(L[b])
        a = float((c == cls0).mean())
        agree.append((int(sm[b]), round(max(a, 1 - a), 3), round(a, 3)))
    agree.sort()
    print(json.dumps({"agreement_with_sm0 (sm, max(a,1-a), a)": agree[:40]}))
    same = sum(1 for _, _, a in agree if a > 0.9)
    flip = sum(1 for _, _, a in agree if a < 0.1)
    print(json.dumps({"blocks_same_die_as_block0": same, "blocks_other_die": flip,
                      "unclear": len(agree) - same - flip}))


if __name__ == "__main__":
    main()
