"""Kernel tuning / profiling driver for the u64 query kernel (not part of the product).

  python tools/tune.py --config 3 [--sweep default|full] [--ncu]

Builds the config's index with the reference builder (cached in /dev/shm for the call),
generates the shuffled query stream on the device, then times the query kernel under
launch-shape / L2 / compile-variant settings. --ncu runs exactly one query launch after
setup (for `ncu -k regex:k_query_u64 -c 1`).
"""
import argparse
import ctypes as C
import glob
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import CONFIGS, GEN_SEED, PERM_SEED, SAMPLE_SEED, ref_params  # noqa: E402
from oracle.bindings import Ref  # noqa: E402

PKG = os.path.join(ROOT, "paper_2502_15539_b200")
u8p = C.POINTER(C.c_uint8)


def load_lib(path):
    L = C.CDLL(path)
    L.ph_gpu_index_create.argtypes = [u8p, C.c_size_t, C.c_int, C.POINTER(C.c_void_p)]
    L.ph_gpu_query_u64.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_int,
                                   C.c_int, C.c_void_p]
    L.ph_gpu_set_launch.argtypes = [C.c_int, C.c_int]
    L.ph_gpu_last_error.restype = C.c_char_p
    return L


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--sweep", default="default")
    ap.add_argument("--ncu", action="store_true")
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    n = cfg["n"]
    bench = C.CDLL(os.path.join(PKG, "libph_bench.so"))
    bench.phb_set_persist.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_float, C.c_size_t]
    bench.phb_max_persist_bytes.restype = C.c_longlong
    bench.phb_get_l2_fetch_granularity.restype = C.c_longlong
    stream = torch.cuda.current_stream()
    sp = C.c_void_p(stream.cuda_stream)

    cache = f"/dev/shm/ph_tune_{n}.ptrh"
    if os.path.exists(cache):
        ptrh = open(cache, "rb").read()
    else:
        keys = torch.empty(n, dtype=torch.int64, device="cuda")
        bench.phb_gen_corpus(C.c_void_p(keys.data_ptr()), C.c_uint64(0), C.c_uint64(n),
                             C.c_uint64(GEN_SEED), sp)
        kh = keys.cpu().numpy().view(np.uint64)
        del keys
        ref = Ref()
        t = time.time()
        ptrh = ref.build_u64(kh, ref_params(ref))
        print(f"# reference build {time.time() - t:.1f}s", file=sys.stderr)
        del kh
        open(cache, "wb").write(ptrh)
    q = torch.empty(n, dtype=torch.int64, device="cuda")
    fn = bench.phb_gen_queries_perm if cfg["order"] == "perm" else bench.phb_gen_queries_sample
    fn(C.c_void_p(q.data_ptr()), C.c_uint64(0), C.c_uint64(n), C.c_uint64(n),
       C.c_uint64(GEN_SEED), C.c_uint64(PERM_SEED if cfg["order"] == "perm" else SAMPLE_SEED), sp)
    out = torch.empty(n, dtype=torch.int32, device="cuda")
    buf = (C.c_uint8 * len(ptrh)).from_buffer_copy(ptrh)

    libs = {"main": os.path.join(PKG, "libph_gpu.so")}
    for p in sorted(glob.glob(os.path.join(PKG, "variants", "libph_gpu_*.so"))):
        libs[os.path.basename(p)[10:-3]] = p
    handles = {}
    for name, p in libs.items():
        L = load_lib(p)
        h = C.c_void_p()
        assert L.ph_gpu_index_create(C.cast(buf, u8p), len(ptrh), 0, C.byref(h)) == 0, \
            L.ph_gpu_last_error()
        handles[name] = (L, h)
    ref_out = None

    def run(name, minimal=1):
        L, h = handles[name]
        rc = L.ph_gpu_query_u64(h, C.c_void_p(q.data_ptr()), n, C.c_void_p(out.data_ptr()), 4,
                                minimal, sp)
        assert rc == 0, L.ph_gpu_last_error()

    if args.ncu:
        run("main")
        torch.cuda.synchronize()
        return

    run("main")
    torch.cuda.synchronize()
    ref_out = out.clone()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    pilots_ptr = None

    def measure(name, minimal=1):
        for _ in range(3):
            run(name, minimal)
        ts = []
        for _ in range(args.reps):
            flush.zero_()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            run(name, minimal)
            b.record(stream)
            b.synchronize()
            ts.append(a.elapsed_time(b))
        if minimal:
            assert torch.equal(out, ref_out), f"variant {name} output differs"
        ts.sort()
        return ts[len(ts) // 2], ts[0]

    results = []

    def rec(tag, **kw):
        med, best = measure(kw.pop("lib", "main"), kw.pop("minimal", 1))
        r = {"tag": tag, "ms_median": round(med, 4), "ms_best": round(best, 4),
             "gkeys_s": round(n / med / 1e6, 2)}
        results.append(r)
        print(json.dumps(r), flush=True)

    print(f"# l2 fetch granularity default: {bench.phb_get_l2_fetch_granularity()} B; "
          f"max persisting L2: {bench.phb_max_persist_bytes() / 2**20:.1f} MiB", flush=True)
    rec("baseline")
    rec("nonminimal", minimal=0)
    for L_, _ in handles.values():
        L_.ph_gpu_set_defer_min.argtypes = [C.c_uint64]
        L_.ph_gpu_set_defer_min(2**64 - 1)
    rec("inline remap (deferral off)")
    for L_, _ in handles.values():
        L_.ph_gpu_set_defer_min(1 << 20)
    for reg in (1, 2):
        for L_, _ in handles.values():
            if hasattr(L_, "ph_gpu_set_regime"):
                L_.ph_gpu_set_regime(reg)
        rec(f"regime={reg}")
    for L_, _ in handles.values():
        if hasattr(L_, "ph_gpu_set_regime"):
            L_.ph_gpu_set_regime(0)
    for name in libs:
        if name != "main":
            rec(f"lib={name}", lib=name)
    for threads, bps in ((128, 4), (128, 8), (64, 16)):
        for L, _ in handles.values():
            L.ph_gpu_set_launch(threads, bps)
        rec(f"launch threads={threads} bps={bps}")
    for L, _ in handles.values():
        L.ph_gpu_set_launch(0, 0)
    L, h = handles["main"]
    L.ph_gpu_index_set_l2_policy.argtypes = [C.c_void_p, C.c_uint64, C.c_int]
    for flags in ((0, 1, 2, 3) if args.sweep in ("full", "l2") else ()):
        for hot_mb in ((16, 32, 48, 64, 79, 96, 128) if args.sweep == "full" else (32, 64, 79)):
            assert L.ph_gpu_index_set_l2_policy(h, hot_mb << 20, flags) == 0
            rec(f"l2 hot_mb={hot_mb} flags={flags}")
    assert L.ph_gpu_index_set_l2_policy(h, 1 << 40, 2) == 0
    rec("l2 identity layout, no window")
    L.ph_gpu_index_set_l2_policy(h, 64 << 20, 0)
    print(json.dumps({"summary": results}))


if __name__ == "__main__":
    main()
