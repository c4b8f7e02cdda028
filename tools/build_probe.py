"""Times ph_gpu_build_u64 at a config's n with the pilot search on the GPU and on host threads
(not the product). PH_GPU_BUILD_TRACE=1 prints the GPU search's stage times.

  python tools/build_probe.py [--n 1000000000] [--modes 2,1]
"""
import argparse
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_000_000_000)
    ap.add_argument("--modes", default="2")
    ap.add_argument("--lam", type=int, default=30)
    ap.add_argument("--host-keys", action="store_true", help="keys in (pageable) host memory")
    a = ap.parse_args()
    from oracle.bindings import corpus_u64_np
    from paper_2502_15539_b200 import ph_gpu
    os.environ["PH_GPU_BUILD_TRACE"] = "1"
    keys = corpus_u64_np(0, a.n, 42)
    if not a.host_keys:
        keys = torch.from_numpy(keys.view("int64")).cuda()
    bp = ph_gpu.build_params("default", lambda_=(a.lam, 10))
    outs = []
    for m in [int(x) for x in a.modes.split(",")]:
        ph_gpu.set_build_search(m)
        t = time.time()
        b, st = ph_gpu.build_u64(keys, bp, stats=True)
        dt = time.time() - t
        outs.append(b)
        print(f"mode {m}: {dt:.2f} s, search {st['search_ms']:.0f} ms, prepare {st['prepare_ms']:.0f} ms, "
              f"remap {st['remap_ms']:.0f} ms, upload {st['upload_ms']:.0f} ms, evictions {st['total_evictions']}, gpu {st['search_on_gpu']}",
              flush=True)
    assert all(o == outs[0] for o in outs)


if __name__ == "__main__":
    main()
