"""Builds the native libraries in-tree with nvcc for sm_100a (no JIT cache).

  paper_2502_15539_b200/libph_gpu.so    the product: query kernels + C ABI (include/ph_gpu.h)
  paper_2502_15539_b200/libph_bench.so  measurement tools: roofline microbenchmarks and
                                        device-side synthetic query-stream generators
  tests/cpp/test_query_gpu              C++ test driving the C++ wrapper (include/ph_gpu/index.hpp)

Run: python -m paper_2502_15539_b200.build  (or __graft_entry__.build()).
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr", "-Xptxas", "-v",
           "-Xcompiler", "-fPIC,-O3", "-cudart", "static"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _run(cmd, log):
    r = subprocess.run(cmd, capture_output=True, text=True)
    with open(log, "a") as f:
        f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr + "\n")
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"build failed: {' '.join(cmd)}")


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build_lib(name, sources, extra=(), log=None, force=False):
    out = os.path.join(PKG, name)
    hdrs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    hdrs.append(os.path.join(ROOT, "include", "ph_gpu.h"))
    srcs = [os.path.join(CSRC, s) for s in sources]
    if not force and not _stale(out, srcs + hdrs):
        return out
    objdir = os.path.join(PKG, "build", os.path.basename(name)[:-3])
    os.makedirs(objdir, exist_ok=True)
    objs = [os.path.join(objdir, os.path.basename(s) + ".o") for s in srcs]
    from concurrent.futures import ThreadPoolExecutor  # one nvcc per source, in parallel
    with ThreadPoolExecutor(max_workers=max(1, min(len(srcs), os.cpu_count() or 1))) as ex:
        futs = [ex.submit(_run, [nvcc(), *ARCH, *NVFLAGS, *extra, "-I", CSRC, "-I",
                                 os.path.join(ROOT, "include"), "-c", s, "-o", o], log)
                for s, o in zip(srcs, objs)]
        for f in futs:
            f.result()
    _run([nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", out, *objs], log)
    return out


def build_cpp_test(log):
    src = os.path.join(ROOT, "tests", "cpp", "test_query_gpu.cpp")
    if not os.path.exists(src):
        return None
    out = os.path.join(ROOT, "tests", "cpp", "test_query_gpu")
    deps = [src, os.path.join(ROOT, "include", "ph_gpu.h"),
            os.path.join(ROOT, "include", "ph_gpu", "index.hpp"), os.path.join(PKG, "libph_gpu.so")]
    if _stale(out, deps):
        _run(["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"),
              src, "-o", out, "-L", PKG, "-lph_gpu", f"-Wl,-rpath,{PKG}", "-ldl", "-pthread"], log)
    return out


PRODUCT_SOURCES = ["ph_query.cu", "ph_query_bytes.cu", "ph_partition.cu", "ph_build.cu", "ph_sort.cu",
                   "ph_builder.cu", "ph_search.cu", "ph_abi.cu"]


def build_variants(defs, log=None, force=False):
    """Tuning builds of the product with different compile-time knobs (tools/tune.py)."""
    os.makedirs(os.path.join(PKG, "variants"), exist_ok=True)
    outs = []
    for name, flags in defs.items():
        out = build_lib(os.path.join("variants", f"libph_gpu_{name}.so"),
                        PRODUCT_SOURCES, extra=flags, log=log,
                        force=force)
        outs.append(out)
    return outs


def main(force=False):
    log = os.path.join(PKG, "build", "build.log")
    os.makedirs(os.path.dirname(log), exist_ok=True)
    open(log, "w").close()
    libs = [
        build_lib("libph_gpu.so", PRODUCT_SOURCES, log=log,
                  force=force),
        build_lib("libph_bench.so", ["ph_bench.cu"], log=log, force=force),
    ]
    t = build_cpp_test(log)
    return libs + ([t] if t else [])


if __name__ == "__main__":
    for p in main(force="--force" in sys.argv):
        print(p)
