"""GPU parity tests: the sm_100a query kernels (through the C ABI) against the reference.

The reference answers come from (a) the committed golden fixtures (made by the reference
library, tests/golden/gen_golden.py) and (b) the compiled reference library itself
(oracle/_ref/libptrhash_ref.so), which also builds the indexes. Bar: bit-exact, every key.
Mirrors test_query.cpp:23-117, test_construction.cpp:277-320, test_serde.cpp:119-132 and the
acceptance criterion 6 (mode equivalence, acceptance.cpp:253-284).
"""
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT, golden_names, load_golden

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

THREADS = os.cpu_count() or 8


@pytest.fixture(scope="module")
def ph():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2502_15539_b200 import ph_gpu
    return ph_gpu


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).cuda()


def host_u(t, width):
    return t.cpu().numpy().view(np.uint32 if width == 4 else np.uint64)


def concat(strs):
    offs = np.zeros(len(strs) + 1, dtype=np.uint64)
    offs[1:] = np.cumsum([len(s) for s in strs])
    data = np.frombuffer(b"".join(strs) or b"\0", dtype=np.uint8).copy()
    return data, offs


def gpu_query(idx, q, minimal, width):
    out = idx.query(dev(q), minimal=minimal, out_width=width)
    torch.cuda.synchronize()
    return host_u(out, width).astype(np.uint64)


@pytest.mark.parametrize("name", golden_names())
def test_golden_fixtures(ph, name):
    ptrh, rec = load_golden(name)
    idx = ph.PtrHashIndex(ptrh)
    before = ph.launch_count()
    for minimal, key in ((True, "minimal"), (False, "nonminimal")):
        want = np.array(rec[key], dtype=np.uint64)
        for width in (4, 8):
            if "queries" in rec:
                q = np.array(rec["queries"], dtype=np.uint64)
                got_dev = gpu_query(idx, q, minimal, width)
                got_host = idx.query(q, minimal=minimal, out_width=width).astype(np.uint64)
            else:
                data, offs = concat([bytes.fromhex(h) for h in rec["queries_hex"]])
                out = idx.query((torch.from_numpy(data).cuda(),
                                 torch.from_numpy(offs.view(np.int64)).cuda()),
                                minimal=minimal, out_width=width)
                torch.cuda.synchronize()
                got_dev = host_u(out, width).astype(np.uint64)
                got_host = idx.query((data, offs), minimal=minimal, out_width=width).astype(np.uint64)
            assert np.array_equal(got_dev, want), (name, minimal, width)
            assert np.array_equal(got_host, want), (name, minimal, width)
    assert ph.launch_count() > before  # the native kernels ran


def test_golden_single_key(ph):
    for name in ("default_l30", "quadratic_ef", "shape_one_slot", "str_default"):
        ptrh, rec = load_golden(name)
        idx = ph.PtrHashIndex(ptrh)
        for i in range(0, len(rec["minimal"]), max(1, len(rec["minimal"]) // 25)):
            key = (int(rec["queries"][i]) if "queries" in rec
                   else bytes.fromhex(rec["queries_hex"][i]))
            assert idx.index(key) == rec["minimal"][i]
            assert idx.index_no_remap(key) == rec["nonminimal"][i]


CASES = [
    ("default", {"lambda_": (30, 10)}),          # the BASELINE configs' parameters
    ("fast", {}), ("compact", {}),
    ("default", {"remap": "plain32"}),
    ("default", {"remap": "elias-fano"}),
    ("default", {"bucket_fn": "linear"}),
    ("default", {"bucket_fn": "quadratic"}),
    ("default", {"bucket_fn": "skewed"}),
    ("default", {"bucket_fn": "optimal"}),
    ("default", {"reduce": "pow2-mul"}),
    ("default", {"reduce": "fastmod-single", "remap": "plain32"}),
]


@pytest.mark.parametrize("preset,over", CASES, ids=[f"{p}-{o}" for p, o in CASES])
def test_fresh_index_vs_reference(ph, ref, preset, over):
    from oracle.bindings import corpus_u64_np
    n = 300_000
    keys = corpus_u64_np(0, n, 21)
    ptrh = ref.build_u64(keys, ref.params(preset, **over))
    ri = ref.load(ptrh)
    idx = ph.PtrHashIndex(ptrh)
    q = np.concatenate([keys, corpus_u64_np(0, n // 2, 22)])  # members + non-members
    for minimal in (True, False):
        want = ri.query_u64(q, minimal, "loop", threads=THREADS)
        for width in (4, 8):
            assert np.array_equal(gpu_query(idx, q, minimal, width), want)
    got = gpu_query(idx, keys, True, 4)
    assert np.array_equal(np.sort(got), np.arange(n, dtype=np.uint64))


@pytest.mark.parametrize("slots_target", [6000, 9000, 300_000, 2_200_000])
def test_mod_fast_and_64bit_reduce_agree(ph, ref, slots_target, monkeypatch):
    """y mod S by the 32-bit form (ph_arith.cuh mod_fast, 2^13 <= S < 2^21) and by the 64-bit
    form (PH_GPU_NO_MODFAST) on the same index: both equal the reference (reduce.hpp:38-43).
    S straddles the fast form's range (one part of ~slots_target slots)."""
    from oracle.bindings import corpus_u64_np
    n = int(slots_target * 0.99)
    keys = corpus_u64_np(0, n, 31)
    S = slots_target
    ptrh = ref.build_u64_shape(keys, ref.params("default", lambda_=(30, 10)), 1, S,
                               max(1, n // 3))
    ri = ref.load(ptrh)
    q = np.concatenate([keys, corpus_u64_np(0, n, 32)])
    outs = []
    for off in ("", "1"):
        if off:
            monkeypatch.setenv("PH_GPU_NO_MODFAST", off)
        idx = ph.PtrHashIndex(ptrh)
        outs.append([gpu_query(idx, q, m, 8) for m in (True, False)])
        idx.close()
    for m, got_fast, got_slow in zip((True, False), outs[0], outs[1]):
        want = ri.query_u64(q, m, "loop", threads=THREADS)
        assert np.array_equal(got_fast, want) and np.array_equal(got_slow, want)


def test_config1_full_bijective_and_bitexact(ph, ref):
    """BASELINE config 1: n=1e7, λ=3.0, α=0.99, cubic, CacheLineEF, shuffled, u32 out."""
    from oracle.bindings import corpus_u64_np
    import ctypes as C
    n = 10_000_000
    keys = corpus_u64_np(0, n, 42)
    ptrh = ref.build_u64(keys, ref.params("default", lambda_=(30, 10)))
    ri = ref.load(ptrh)
    idx = ph.PtrHashIndex(ptrh)
    assert idx.info.remap_kind == 1 and idx.info.bucket_fn == 2 and not idx.info.pow2
    bench = C.CDLL(os.path.join(ROOT, "paper_2502_15539_b200", "libph_bench.so"))
    q = torch.empty(n, dtype=torch.int64, device="cuda")
    assert bench.phb_gen_queries_perm(C.c_void_p(q.data_ptr()), C.c_uint64(0), C.c_uint64(n),
                                      C.c_uint64(n), C.c_uint64(42), C.c_uint64(7), None) == 0
    qh = q.cpu().numpy().view(np.uint64)
    assert np.array_equal(np.sort(qh), np.sort(keys))  # a permutation of the key set
    for minimal in (True, False):
        out = idx.query(q, minimal=minimal, out_width=4)
        torch.cuda.synchronize()
        got = host_u(out, 4).astype(np.uint64)
        want = ri.query_u64(qh, minimal, "stream", 32, threads=THREADS)
        assert np.array_equal(got, want)
        if minimal:
            bits = torch.zeros((n + 31) // 32, dtype=torch.int32, device="cuda")
            bad = torch.zeros(2, dtype=torch.int64, device="cuda")
            bench.phb_bijection(C.c_void_p(out.data_ptr()), C.c_uint64(n), C.c_uint64(n),
                                C.c_void_p(bits.data_ptr()), C.c_void_p(bad.data_ptr()), None)
            assert bad.tolist() == [0, 0]


@pytest.mark.parametrize("count", [0, 1, 2, 31, 32, 33, 255, 256, 257, 1000, 4097])
def test_ragged_and_empty(ph, ref, count):
    ptrh, rec = load_golden("default_l30")
    idx = ph.PtrHashIndex(ptrh)
    q = np.array(rec["queries"][:count], dtype=np.uint64)
    want = np.array(rec["minimal"][:count], dtype=np.uint64)
    if count == 0:
        out = torch.empty(0, dtype=torch.int32, device="cuda")
        idx.query(torch.empty(0, dtype=torch.int64, device="cuda"), out=out, out_width=4)
        assert idx.query(q, out_width=8).size == 0
        return
    assert np.array_equal(gpu_query(idx, q, True, 4), want)
    assert np.array_equal(idx.query(q, out_width=8), want)


def test_unaligned_device_pointers(ph):
    ptrh, rec = load_golden("fast")
    idx = ph.PtrHashIndex(ptrh)
    q = np.array(rec["queries"], dtype=np.uint64)
    want = np.array(rec["minimal"], dtype=np.uint64)
    big = dev(np.concatenate([np.zeros(1, dtype=np.uint64), q]))
    out = torch.zeros(q.size + 1, dtype=torch.int32, device="cuda")
    idx.query(big[1:], out=out[1:], out_width=4)
    torch.cuda.synchronize()
    assert np.array_equal(host_u(out, 4)[1:].astype(np.uint64), want)


def test_concurrent_streams_share_one_index(ph):
    ptrh, rec = load_golden("default_l30")
    idx = ph.PtrHashIndex(ptrh)
    q = dev(np.array(rec["queries"] * 50, dtype=np.uint64))
    want = np.array(rec["minimal"] * 50, dtype=np.uint64)
    streams = [torch.cuda.Stream() for _ in range(4)]
    outs = []
    for s in streams:
        with torch.cuda.stream(s):
            outs.append(idx.query(q, out_width=8))
    torch.cuda.synchronize()
    for o in outs:
        assert np.array_equal(host_u(o, 8), want)


def test_host_path_pinned_and_pageable(ph, ref):
    from oracle.bindings import corpus_u64_np
    n = 20_000_000  # > 2 pipeline chunks
    keys = corpus_u64_np(0, 1_000_000, 31)
    ptrh = ref.build_u64(keys, ref.params("default", lambda_=(30, 10)))
    idx = ph.PtrHashIndex(ptrh)
    q = corpus_u64_np(0, n, 32)
    q[: keys.size] = keys
    want = gpu_query(idx, q, True, 4)
    pageable = idx.query(q, out_width=4)
    assert np.array_equal(pageable.astype(np.uint64), want)
    pin_q = torch.from_numpy(q.view(np.int64)).pin_memory()
    pin_o = torch.empty(n, dtype=torch.int32).pin_memory()
    idx.query(pin_q, out=pin_o, out_width=4)
    assert np.array_equal(pin_o.numpy().view(np.uint32).astype(np.uint64), want)


def test_string_keys_vs_reference(ph, ref):
    """config-4 style strings (len U[8,64], printable ASCII) plus edge lengths."""
    from oracle.bindings import string_corpus
    strs = string_corpus(100_000, 77)
    data, offs = concat(strs)
    ptrh = ref.build_bytes(data, offs, ref.params("default", lambda_=(30, 10)), lean=True)
    ri = ref.load(ptrh)
    idx = ph.PtrHashIndex(ptrh)
    extra = [b"", b"a", b"x" * 16, b"y" * 17, b"z" * 200, bytes(range(256)) * 4]
    allq = strs + string_corpus(5000, 78, 0, 100) + extra
    d2, o2 = concat(allq)
    for minimal in (True, False):
        want = ri.query_bytes(d2, o2, minimal, "single", threads=THREADS)
        for width in (4, 8):
            out = idx.query((torch.from_numpy(d2).cuda(), torch.from_numpy(o2.view(np.int64)).cuda()),
                            minimal=minimal, out_width=width)
            torch.cuda.synchronize()
            assert np.array_equal(host_u(out, width).astype(np.uint64), want)
        assert np.array_equal(idx.query((d2, o2), minimal=minimal, out_width=8), want)
    got = idx.query((data, offs), out_width=4).astype(np.uint64)
    assert np.array_equal(np.sort(got), np.arange(len(strs), dtype=np.uint64))


def test_key_kind_mismatch_is_an_error(ph):
    ptrh, _ = load_golden("str_default")
    idx = ph.PtrHashIndex(ptrh)
    with pytest.raises(ph.PhGpuError):
        idx.query(np.arange(10, dtype=np.uint64))
    ptrh, _ = load_golden("fast")
    idx = ph.PtrHashIndex(ptrh)
    with pytest.raises(ph.PhGpuError):
        idx.index(b"abc")


def test_cpp_wrapper_suite():
    exe = os.path.join(ROOT, "tests", "cpp", "test_query_gpu")
    so = os.path.join(ROOT, "oracle", "_ref", "libptrhash_ref.so")
    r = subprocess.run([exe, so], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stderr


# ---- fused k-mer front end (BASELINE config 5) ----

@pytest.mark.parametrize("k,n_bases", [(31, 200_030), (31, 64_000), (32, 50_017), (16, 40_001),
                                       (5, 3_001), (1, 100), (31, 31), (31, 30)])
def test_kmers_fused_vs_reference(ph, ref, port, k, n_bases):
    seq = port.gen_dna(n_bases, 44 + k)
    kmers = port.kmers(seq, n_bases, k)
    if kmers.size == 0:
        ptrh, _ = load_golden("default_l30")
        idx = ph.PtrHashIndex(ptrh)
        assert idx.query_kmers(seq, n_bases, k).size == 0
        return
    uniq = np.unique(kmers)
    ptrh = ref.build_u64(uniq, ref.params("default", lambda_=(30, 10)))
    ri = ref.load(ptrh)
    idx = ph.PtrHashIndex(ptrh)
    for minimal in (True, False):
        want = ri.query_u64(kmers, minimal, "stream", 32, threads=THREADS)
        d_seq = torch.from_numpy(seq.view(np.int64)).cuda()
        got = idx.query_kmers(d_seq, n_bases, k, minimal=minimal, out_width=8)
        torch.cuda.synchronize()
        assert np.array_equal(host_u(got, 8), want)
        got_h = idx.query_kmers(seq, n_bases, k, minimal=minimal, out_width=4)
        assert np.array_equal(got_h.astype(np.uint64), want)
        # identical to materialising the k-mers and querying them as u64 keys
        assert np.array_equal(gpu_query(idx, kmers, minimal, 4), want)


def test_kmer_harness_matches_oracle(port):
    import ctypes as C
    bench = C.CDLL(os.path.join(ROOT, "paper_2502_15539_b200", "libph_bench.so"))
    n_bases = 100_003
    seq = port.gen_dna(n_bases, 44)
    d_seq = torch.empty(seq.size, dtype=torch.int64, device="cuda")
    bench.phb_gen_dna(C.c_void_p(d_seq.data_ptr()), C.c_uint64(seq.size), C.c_uint64(44), None)
    assert np.array_equal(d_seq.cpu().numpy().view(np.uint64), seq)
    for k in (31, 32, 7):
        out = torch.empty(n_bases - k + 1, dtype=torch.int64, device="cuda")
        bench.phb_kmers(C.c_void_p(d_seq.data_ptr()), C.c_uint64(n_bases), k,
                        C.c_void_p(out.data_ptr()), None)
        assert np.array_equal(host_u(out, 8), port.kmers(seq, n_bases, k))


def test_load_from_file_matches_create(ph, tmp_path):
    """ph_gpu_index_load (load_index, serde.cpp:251-260) == create from the same bytes."""
    for name in ("default_l30", "quadratic_ef", "str_default"):
        ptrh, rec = load_golden(name)
        path = tmp_path / f"{name}.ptrh"
        path.write_bytes(ptrh)
        idx = ph.PtrHashIndex.load(str(path))
        assert idx.shape() == ph.PtrHashIndex(ptrh).shape()
        if "queries" in rec:
            q = np.array(rec["queries"], dtype=np.uint64)
            assert np.array_equal(gpu_query(idx, q, True, 8), np.array(rec["minimal"], np.uint64))
    bad = tmp_path / "bad.ptrh"
    bad.write_bytes(b"PTRX" + bytes(80))
    with pytest.raises(ph.SerdeError):
        ph.PtrHashIndex.load(str(bad))
    with pytest.raises(ph.PhGpuError):
        ph.PtrHashIndex.load(str(tmp_path / "missing.ptrh"))


def test_verify_bijection_on_device(ph, ref):
    """ph_gpu_verify_bijection (verify_bijection, ptrhash.cpp:186-210): 0/0 on a real
    answer, and it counts planted out-of-range values and duplicates."""
    from oracle.bindings import corpus_u64_np
    n = 200_000
    keys = corpus_u64_np(0, n, 31)
    idx = ph.PtrHashIndex(ref.build_u64(keys, ref.params("default")))
    for width in (4, 8):
        out = idx.query(dev(keys), minimal=True, out_width=width)
        assert idx.verify_bijection(out) == (0, 0)
        bad = out.clone()
        bad[5] = n + 3        # out of range
        bad[7] = bad[8]       # one duplicate
        bad[9] = bad[8]       # another
        assert idx.verify_bijection(bad) == (1, 2)
    nm = idx.query(dev(keys), minimal=False, out_width=8)
    P, S = idx.shape()[1:3]
    assert idx.verify_bijection(nm, n=P * S) == (0, 0)


@pytest.mark.parametrize("hot_bytes,flags", [(0, 0), (0, 2), (4096, 0), (4096, 1), (4096, 2),
                                             (1 << 16, 3)])
def test_pilot_layouts_bitexact(ph, ref, hot_bytes, flags):
    """ph_gpu_index_set_l2_policy: the hot-first layout (hot region of hot_bytes, with and
    without the persisting window / evict_first cold loads) and the file order answer
    identically to the reference, through the direct kernels and (file order) the
    partitioned path, for u64 keys and k-mers."""
    from oracle.bindings import corpus_u64_np
    n = 300_000
    keys = corpus_u64_np(0, n, 71)
    ptrh = ref.build_u64(keys, ref.params("default", lambda_=(30, 10)))
    ri = ref.load(ptrh)
    idx = ph.PtrHashIndex(ptrh)
    idx.set_l2_policy(hot_bytes, flags)
    q = np.concatenate([keys, corpus_u64_np(0, n // 3, 72)])
    for minimal in (True, False):
        want = ri.query_u64(q, minimal, "loop", threads=THREADS)
        for width in (4, 8):
            assert np.array_equal(gpu_query(idx, q, minimal, width), want), (minimal, width)
    if hot_bytes == 0:  # file order: the partitioned path applies
        ph.set_partition(2)
        try:
            assert np.array_equal(gpu_query(idx, q, True, 4),
                                  ri.query_u64(q, True, "loop", threads=THREADS))
        finally:
            ph.set_partition(0)
    idx.set_l2_policy(64 << 20, 0)  # back to the default of an L2-sized pilot array
    assert np.array_equal(gpu_query(idx, keys, True, 8),
                          ri.query_u64(keys, True, "loop", threads=THREADS))
