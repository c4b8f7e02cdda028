"""e2e (host API) timing on a bench.py workload, per pipeline chunk size and pilot layout
(not part of the product).

  python tools/e2e_probe.py --config 3 [--chunks 4194304,8388608,...] [--layouts default,file]
"""
import argparse
import ctypes as C
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


class _Dist:
    world, rank, local = 1, 0, 0

    def barrier(self):
        pass


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--chunks", default="8388608")
    ap.add_argument("--layouts", default="default,file")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--sampler", action="store_true", help="run bench.py's NVML clock sampler")
    ap.add_argument("--device-first", action="store_true")
    a = ap.parse_args()
    cfg = dict(bench.CONFIGS[a.config])
    cfg.pop("layout", None)
    lib = C.CDLL(os.path.join(ROOT, "paper_2502_15539_b200", "libph_bench.so"))
    stream = torch.cuda.current_stream()
    W = bench.WORKLOADS[cfg["kind"]](a, cfg, _Dist(), lib, C.c_void_p(stream.cuda_stream))
    pin_o = torch.empty(W.nq, dtype=torch.int32).pin_memory()
    if a.sampler:
        bench.ClockSampler(0).start()
    if a.device_first:  # as bench.py does: device-resident queries (partitioned path) first
        out = torch.empty(W.nq, dtype=torch.int32, device="cuda")
        for _ in range(3):
            W.query(out, True, stream.cuda_stream)
        torch.cuda.synchronize()
    for layout in a.layouts.split(","):
        if layout == "file":
            W.idx.set_l2_policy(0, 2)
        else:
            W.idx.set_l2_policy(64 << 20, 0)
        for ck in a.chunks.split(","):
            os.environ["PH_GPU_CHUNK_KEYS"] = ck
            W.e2e(pin_o)
            best, ts = 1e9, []
            for _ in range(a.reps):
                torch.cuda.synchronize()
                t = time.perf_counter()
                W.e2e(pin_o)
                torch.cuda.synchronize()
                ts.append(round((time.perf_counter() - t) * 1e3, 1))
                best = min(best, ts[-1] / 1e3)
            print(json.dumps({"config": a.config, "layout": layout, "chunk_keys": int(ck),
                              "sampler": a.sampler,
                              "ms": round(best * 1e3, 1), "all_ms": ts,
                              "e2e_gkeys_s": round(W.nq / best / 1e9, 3)}), flush=True)


if __name__ == "__main__":
    main()
