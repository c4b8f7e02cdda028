"""B200-native (sm_100a) PtrHash query path (arXiv 2502.15539).

The product is ``libph_gpu.so`` (CUDA kernels + the C ABI in include/ph_gpu.h).
``paper_2502_15539_b200.ph_gpu`` is its Python mirror of the reference's
``PtrHashIndex`` query API; importing it fails loudly if the library is missing.
"""
import os

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_GPU = os.path.join(PKG_DIR, "libph_gpu.so")
LIB_BENCH = os.path.join(PKG_DIR, "libph_bench.so")
