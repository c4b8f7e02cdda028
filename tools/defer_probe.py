"""Direct L2-regime kernel at configs 1/2 shapes (synthetic index, tools/synth_perf.py):
deferred remap (warp lists + k_remap_patch) vs inline warp-compacted remap. Timing only."""
import ctypes as C
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from tools.synth_perf import SHAPES, synth_ptrh  # noqa: E402


def main():
    from paper_2502_15539_b200 import ph_gpu
    L = ph_gpu._L
    L.ph_gpu_set_defer_min.argtypes = [C.c_uint64]
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    for cfg in (1, 2):
        idx = ph_gpu.PtrHashIndex(synth_ptrh(cfg))
        n = SHAPES[cfg][0]
        g = torch.Generator(device="cuda")
        g.manual_seed(7)
        keys = torch.randint(-2**63, 2**63 - 1, (n,), dtype=torch.int64, device="cuda", generator=g)
        out = torch.empty(n, dtype=torch.int32, device="cuda")
        res = {}
        for name, dm in (("deferred", 1 << 20), ("inline", 2**64 - 1)):
            L.ph_gpu_set_defer_min(dm)
            idx.query(keys, out=out, minimal=True, out_width=4)
            ts = []
            for _ in range(20):
                flush.fill_(1)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                idx.query(keys, out=out, minimal=True, out_width=4)
                b.record()
                b.synchronize()
                ts.append(a.elapsed_time(b))
            ts.sort()
            res[name] = out.clone()
            print(f"config {cfg} remap {name:8s}: best {ts[0]:.4f} ms median {ts[len(ts) // 2]:.4f} ms "
                  f"{n / ts[0] / 1e6:.1f} Gkeys/s", flush=True)
        assert torch.equal(res["deferred"], res["inline"])
        L.ph_gpu_set_defer_min(1 << 20)


if __name__ == "__main__":
    main()
