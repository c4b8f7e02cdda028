"""Construction assist timing (not the query path): the front phases of one
u64 build attempt at n keys on the GPU (ph_gpu_build_prepare_u64, event-timed, keys
device-resident) against the reference's own code for the same phases on all host cores
(ref_build_prepare_u64: hash_all + scatter_to_parts + per-part std::sort), on a sample.

  python tools/build_assist_bench.py [--n 1000000000] [--cpu-sample 100000000]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=10**9)
    ap.add_argument("--cpu-sample", type=int, default=10**8)
    a = ap.parse_args()
    from oracle.bindings import Ref, corpus_u64_np
    from paper_2502_15539_b200 import ph_gpu
    ref = Ref()
    params = ref.params("default", lambda_=(30, 10))
    P, S, _ = ref.shape(a.n, params)
    seed = 0x9E3779B97F4A7C15
    keys = torch.empty(a.n, dtype=torch.int64, device="cuda")
    step = 1 << 27
    for s in range(0, a.n, step):  # corpus_u64 (corpus.hpp:14-16), generated on the host
        m = min(step, a.n - s)
        keys[s:s + m] = torch.from_numpy(corpus_u64_np(s, m, 42).view(np.int64)).cuda()
    ph_gpu.build_prepare_u64(keys[: 1 << 20], P, S, seed)  # warm-up
    ts = []
    for _ in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        h, off, st = ph_gpu.build_prepare_u64(keys, P, S, seed)  # synchronous
        ts.append(time.perf_counter() - t)
        del h, off
    gpu_ms = min(ts) * 1e3
    m = min(a.cpu_sample, a.n)
    ks = keys[:m].cpu().numpy().view(np.uint64)
    Pm, Sm, _ = ref.shape(m, params)
    t = time.perf_counter()
    _, _, st_c = ref.build_prepare_u64(ks, Pm, Sm, seed, threads=0)
    cpu_s = time.perf_counter() - t
    print(json.dumps({"n": a.n, "parts": P, "gpu_ms": round(gpu_ms, 2),
                      "gpu_ns_per_key": round(gpu_ms * 1e6 / a.n, 4), "status": st,
                      "cpu_sample": m, "cpu_threads": ref.hw_threads(),
                      "cpu_ns_per_key": round(cpu_s * 1e9 / m, 3), "cpu_status": st_c}))


if __name__ == "__main__":
    main()
