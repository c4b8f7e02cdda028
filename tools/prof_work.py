"""Profile driver: set up a bench.py workload (config 1-5) and run the query launch once
(--ncu) or time it (default). Not part of the product.

  python tools/prof_work.py --config 4 [--ncu] [--n N]
"""
import argparse
import ctypes as C
import os
import sys

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
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--ncu", action="store_true")
    ap.add_argument("--n", type=int, default=0, help="override the config's n")
    ap.add_argument("--minimal", type=int, default=1)
    ap.add_argument("--regimes", default="", help="comma list of ph_gpu_set_regime values to time")
    ap.add_argument("--partition", default="", help="comma list of ph_gpu_set_partition modes")
    ap.add_argument("--layout", default="default", help="default | file (pilot layout)")
    ap.add_argument("--no-persist", action="store_true",
                    help="drop the persisting-L2 carve-out after the index is created")
    a = ap.parse_args()
    for k, v in dict(construction=False, verify="none", cpu_sample=0, no_cpu_baseline=True, no_replay=True,
                     secondary_configs=False, steps=1, warmup=0, impl="ours").items():
        if not hasattr(a, k):  # attributes bench.py's workloads read from its own parser
            setattr(a, k, v)
    cfg = dict(bench.CONFIGS[a.config])
    if a.n:
        cfg["n"] = a.n
    lib = C.CDLL(os.path.join(ROOT, "paper_2502_15539_b200", "libph_bench.so"))
    stream = torch.cuda.current_stream()
    W = bench.WORKLOADS[cfg["kind"]](a, cfg, _Dist(), lib, C.c_void_p(stream.cuda_stream))
    out = torch.empty(W.nq, dtype=torch.int32, device="cuda")
    if a.no_persist:
        lib.phb_set_persist.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_float, C.c_size_t]
        assert lib.phb_set_persist(C.c_void_p(stream.cuda_stream), None, 0, 0.0, 0) == 0
    from paper_2502_15539_b200 import ph_gpu
    if a.layout == "file":  # file-order pilots, no persisting window (partition-capable)
        W.idx.set_l2_policy(0, 2)
    if a.ncu and a.partition:  # profile the first listed partition mode
        ph_gpu.set_partition(int(a.partition.split(",")[0]))
    W.query(out, bool(a.minimal), stream.cuda_stream)
    torch.cuda.synchronize()
    if a.ncu:
        return
    from paper_2502_15539_b200 import ph_gpu
    ph_gpu._L.ph_gpu_set_regime.argtypes = [C.c_int]
    ph_gpu._L.ph_gpu_set_partition.argtypes = [C.c_int]
    combos = [(int(r), int(pm)) for r in (a.regimes.split(",") if a.regimes else ["0"])
              for pm in (a.partition.split(",") if a.partition else ["0"])]
    ref_out = None
    for reg, pm in combos:
        ph_gpu._L.ph_gpu_set_regime(reg)
        ph_gpu._L.ph_gpu_set_partition(pm)
        for minimal in (True, False):
            W.query(out, minimal, stream.cuda_stream)
            ts = []
            for _ in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                W.query(out, minimal, stream.cuda_stream)
                e1.record(stream)
                e1.synchronize()
                ts.append(e0.elapsed_time(e1))
            if minimal:
                if ref_out is None:
                    ref_out = out.clone()
                assert torch.equal(out, ref_out), "outputs differ between modes"
            print(f"config {a.config} n={W.nq} regime={reg} partition={pm} minimal={int(minimal)}: best "
                  f"{min(ts):.3f} ms, {W.nq / min(ts) / 1e6:.2f} Gkeys/s", flush=True)


if __name__ == "__main__":
    main()
