"""Timing-only harness on a synthetic index of a bench config's exact shape (not the product,
not a parity test). The PTRH header comes from a small index built by the reference builder
with the same parameters; n, P, S, B are set to the config's shape and the
pilot and CacheLineEF payloads are seeded random bytes. Every kernel path does the same
arithmetic and memory traffic on it as on the real index, so the paths can be timed against
each other in seconds instead of building a 1e9-key index; their outputs must agree.

  python tools/synth_perf.py --config 3 [--paths "direct;v2;v2@PH_GPU_PART_CHUNKS=4"] [--reps 5]

A path is direct | direct_hot | v2 | v3, optionally followed by @NAME=VAL,NAME=VAL (environment
knobs read by the library at call time).
"""
import argparse
import ctypes as C
import os
import struct
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SHAPES = {  # n, P, S, B (reference compute_shape)
    1: (10**7, 26, 388_501, 128_206),
    2: (10**8, 176, 573_922, 189_395),
    3: (10**9, 1326, 761_766, 251_383),
    4: (3 * 10**8, 456, 664_541, 219_299),
}


def synth_ptrh(cfg: int, seed: int = 1) -> bytes:
    from oracle.bindings import Ref, corpus_u64_np
    ref = Ref()
    small = ref.build_u64(corpus_u64_np(0, 50_000, 42), ref.params("default", lambda_=(30, 10)))
    n, P, S, B = SHAPES[cfg]
    hdr = bytearray(small[:72])
    assert hdr[11] == 1, "expected a CacheLineEF header"
    count = P * S - n
    remap_len = (count + 43) // 44 * 64
    struct.pack_into("<QQQQ", hdr, 16, n, P, S, B)
    struct.pack_into("<QQ", hdr, 56, P * B, remap_len)
    rng = np.random.default_rng(seed)
    pil = rng.integers(0, 256, P * B, dtype=np.uint8)
    rem = rng.integers(0, 256, remap_len, dtype=np.uint8)
    return bytes(hdr) + pil.tobytes() + rem.tobytes()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--paths", default="direct;v2;v3")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--nq", type=int, default=0)
    ap.add_argument("--ncu", action="store_true", help="one call per path, no timing")
    a = ap.parse_args()
    from paper_2502_15539_b200 import ph_gpu
    L = ph_gpu._L
    L.ph_gpu_set_partition.argtypes = [C.c_int]
    ptrh = synth_ptrh(a.config)
    n = SHAPES[a.config][0]
    nq = a.nq or n
    g = torch.Generator(device="cuda")
    g.manual_seed(7)
    keys = torch.randint(-2**63, 2**63 - 1, (nq,), dtype=torch.int64, device="cuda", generator=g)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    outs = {}
    base_env = dict(os.environ)
    for path in a.paths.split(";"):
        os.environ.clear()
        os.environ.update(base_env)
        name = path
        if "@" in path:
            name, kv = path.split("@", 1)
            for item in kv.split(","):
                k, v = item.split("=", 1)
                os.environ[k] = v
        if name == "direct_hot":
            idx = ph_gpu.PtrHashIndex(ptrh)  # default layout (hot-first + window)
        else:
            idx = ph_gpu.PtrHashIndex(ptrh)
            idx.set_l2_policy(0, 2)  # file order, no window
        if name in ("v2", "v3"):
            os.environ["PH_GPU_PART_V"] = name[1]
        L.ph_gpu_set_partition(1 if name.startswith("direct") else 2)
        for minimal in (True, False):
            out = torch.empty(nq, dtype=torch.int32, device="cuda")
            idx.query(keys, out=out, minimal=minimal, out_width=4)
            torch.cuda.synchronize()
            if a.ncu:
                continue
            ts = []
            for _ in range(a.reps):
                flush.fill_(1)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                idx.query(keys, out=out, minimal=minimal, out_width=4)
                e1.record()
                e1.synchronize()
                ts.append(e0.elapsed_time(e1))
            outs.setdefault(minimal, {})[path] = out
            ts.sort()
            print(f"config {a.config} {path:40s} minimal={int(minimal)}: best {ts[0]:.3f} ms "
                  f"median {ts[len(ts) // 2]:.3f} ms  {nq / ts[0] / 1e6:.1f} Gkeys/s", flush=True)
        idx.close()
    for minimal, d in outs.items():
        names = list(d)
        for p in names[1:]:
            same = torch.equal(d[names[0]], d[p])
            print(f"minimal={int(minimal)} {names[0]} == {p}: {same}", flush=True)
            assert same


if __name__ == "__main__":
    main()
