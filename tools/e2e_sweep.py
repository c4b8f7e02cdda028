"""e2e (host API) throughput vs pipeline chunk size, config-3-sized key stream (1e9 keys)
against a config-1 index (the e2e path is PCIe-bound; the index size does not matter)."""
import ctypes as C
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.bindings import Ref, corpus_u64_np  # noqa: E402


def main():
    from paper_2502_15539_b200 import ph_gpu
    ref = Ref()
    keys = corpus_u64_np(0, 10_000_000, 42)
    idx = ph_gpu.PtrHashIndex(ref.build_u64(keys, ref.params("default", lambda_=(30, 10))))
    n = 1_000_000_000
    q = torch.empty(n, dtype=torch.int64).pin_memory()
    q.numpy()[:] = np.resize(keys.view(np.int64), n)
    out = torch.empty(n, dtype=torch.int32).pin_memory()
    for ck in (1 << 22, 1 << 23, 1 << 24, 1 << 25, 1 << 26):
        os.environ["PH_GPU_CHUNK_KEYS"] = str(ck)
        idx.query(q, out=out, out_width=4)
        best = 1e9
        for _ in range(3):
            t = time.perf_counter()
            idx.query(q, out=out, out_width=4)
            best = min(best, time.perf_counter() - t)
        print(json.dumps({"chunk_keys": ck, "e2e_gkeys_s": round(n / best / 1e9, 3),
                          "ms": round(best * 1e3, 1)}), flush=True)


if __name__ == "__main__":
    main()
