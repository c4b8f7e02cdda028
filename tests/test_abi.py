"""CPU tests of the C-ABI boundary: the product library loads, exports every entry point
include/ph_gpu.h declares, and rejects malformed PTRH bytes exactly where the reference's
deserialize() does (serde.cpp:176-240) — parse/validation runs before any device work, so
no GPU is needed here."""
import ctypes as C
import os
import re

import pytest

from conftest import ROOT, load_golden

HDR = os.path.join(ROOT, "include", "ph_gpu.h")


def declared_symbols():
    src = open(HDR).read()
    return sorted(set(re.findall(r"\b(ph_gpu_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2502_15539_b200 import ph_gpu  # noqa: F401  (raises if the .so is missing)
    lib = C.CDLL(os.path.join(ROOT, "paper_2502_15539_b200", "libph_gpu.so"))
    syms = declared_symbols()
    assert len(syms) >= 12
    for s in syms:
        assert hasattr(lib, s), s


def test_bench_library_loads():
    lib = C.CDLL(os.path.join(ROOT, "paper_2502_15539_b200", "libph_bench.so"))
    for s in ("phb_gen_queries_perm", "phb_gen_queries_sample", "phb_gather", "phb_bijection"):
        assert hasattr(lib, s)


def test_perm_host_twin_matches_oracle(port):
    lib = C.CDLL(os.path.join(ROOT, "paper_2502_15539_b200", "libph_bench.so"))
    lib.phb_perm_key_host.argtypes = [C.c_uint64] * 4
    lib.phb_perm_key_host.restype = C.c_uint64
    for n in (5, 1000, 10**7):
        for i in (0, 1, n // 2, n - 1):
            want = port.L.pho_corpus_u64(port.L.pho_feistel_perm(i, n, 7), 42)
            assert lib.phb_perm_key_host(i, n, 42, 7) == want


def test_create_rejects_corrupt_ptrh_without_gpu():
    from paper_2502_15539_b200 import ph_gpu
    from test_oracle import _corrupt_cases
    ptrh, _ = load_golden("default_l30")
    for what, bad in _corrupt_cases(ptrh):
        with pytest.raises(ph_gpu.SerdeError):
            ph_gpu.PtrHashIndex(bad)
    with pytest.raises(ph_gpu.SerdeError):
        ph_gpu.PtrHashIndex(b"")


def test_argument_errors():
    from paper_2502_15539_b200 import ph_gpu
    L = ph_gpu._L
    assert L.ph_gpu_index_create(None, 0, 0, None) == ph_gpu.E_INVALID
    assert L.ph_gpu_query_u64(None, None, 0, None, 4, 1, None) == ph_gpu.E_INVALID
    assert L.ph_gpu_set_launch(33, 0) == ph_gpu.E_INVALID
    assert b"multiple of 32" in L.ph_gpu_last_error()
    assert L.ph_gpu_set_launch(0, 0) == ph_gpu.OK
