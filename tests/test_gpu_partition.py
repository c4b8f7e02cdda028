"""GPU tests of the partitioned query path (csrc/ph_partition.cu): forced on for
small indexes (ph_gpu_set_partition(2)), its outputs must equal the reference's for u64
keys and k-mers, u32/u64 outputs, minimal/non-minimal, every bucket function / reduce /
remap encoding of the golden fixtures, and ragged batch sizes."""
import ctypes as C
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
THREADS = os.cpu_count() or 8


@pytest.fixture(scope="module")
def ph():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2502_15539_b200 import ph_gpu
    ph_gpu._L.ph_gpu_set_partition.argtypes = [C.c_int]
    ph_gpu._L.ph_gpu_set_partition(2)
    yield ph_gpu
    ph_gpu._L.ph_gpu_set_partition(0)


@pytest.mark.parametrize("nq", [1, 4095, 4096, 4097, 1_000_003, 3 * (1 << 20) + 17])
def test_partitioned_u64_vs_reference(ph, ref, nq):
    from oracle.bindings import corpus_u64_np
    n = 200_000
    keys = corpus_u64_np(0, n, 61)
    ptrh = ref.build_u64(keys, ref.params("default", lambda_=(30, 10)))
    ri = ref.load(ptrh)
    idx = ph.PtrHashIndex(ptrh)
    q = corpus_u64_np(0, nq, 62)
    m = min(nq, n)
    q[:m] = keys[:m]
    d_q = torch.from_numpy(q.view(np.int64)).cuda()
    before = ph.launch_count()
    for minimal in (True, False):
        want = ri.query_u64(q, minimal, "loop", threads=THREADS)
        for width in (4, 8):
            out = idx.query(d_q, minimal=minimal, out_width=width)
            torch.cuda.synchronize()
            got = out.cpu().numpy().view(np.uint32 if width == 4 else np.uint64).astype(np.uint64)
            assert np.array_equal(got, want), (minimal, width)
    assert ph.launch_count() - before >= 3 * 4  # bin/gather/answer (+ remap lists) per call


def _golden_u64():
    from conftest import golden_names, load_golden
    out = []
    for name in golden_names():
        ptrh, rec = load_golden(name)
        if "queries" in rec:
            out.append(name)
    return out


@pytest.mark.parametrize("name", _golden_u64())
def test_partitioned_golden_fixtures(ph, name):
    """Every u64 golden index (all five bucket functions, pow2 / fastmod S, plain32 /
    CacheLineEF / Elias-Fano remaps, forced shapes) through the partitioned path."""
    from conftest import load_golden
    ptrh, rec = load_golden(name)
    idx = ph.PtrHashIndex(ptrh)
    q = np.array(rec["queries"], dtype=np.uint64)
    q = np.concatenate([q] * 3)  # a few tiles, one partial
    d_q = torch.from_numpy(q.view(np.int64)).cuda()
    for minimal, key in ((True, "minimal"), (False, "nonminimal")):
        want = np.concatenate([np.array(rec[key], dtype=np.uint64)] * 3)
        for width in (4, 8):
            if width == 4 and int(want.max()) >= 1 << 32:
                continue
            out = idx.query(d_q, minimal=minimal, out_width=width)
            torch.cuda.synchronize()
            got = out.cpu().numpy().view(np.uint32 if width == 4 else np.uint64).astype(np.uint64)
            assert np.array_equal(got, want), (name, minimal, width)


def test_partitioned_kmers_vs_reference(ph, ref, port):
    n_bases, k = 2_000_030, 31
    seq = port.gen_dna(n_bases, 45)
    kmers = port.kmers(seq, n_bases, k)
    ptrh = ref.build_u64(np.unique(kmers), ref.params("default", lambda_=(30, 10)))
    ri = ref.load(ptrh)
    idx = ph.PtrHashIndex(ptrh)
    d_seq = torch.from_numpy(seq.view(np.int64)).cuda()
    for minimal in (True, False):
        want = ri.query_u64(kmers, minimal, "stream", 32, threads=THREADS)
        out = idx.query_kmers(d_seq, n_bases, k, minimal=minimal, out_width=4)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy().view(np.uint32).astype(np.uint64), want)


@pytest.mark.parametrize("pattern", ["one_key", "two_keys", "sorted_by_group"])
def test_partitioned_skewed_streams_spill(ph, ref, pattern):
    """Query streams whose groups overflow the per-group regions (pass A's spill region):
    every key identical, two alternating keys, and a stream sorted so whole tiles fall in
    one group. Outputs must still equal the reference's."""
    from oracle.bindings import corpus_u64_np
    n = 200_000
    keys = corpus_u64_np(0, n, 63)
    ptrh = ref.build_u64(keys, ref.params("default", lambda_=(30, 10)))
    ri = ref.load(ptrh)
    idx = ph.PtrHashIndex(ptrh)
    nq = 3_000_017
    if pattern == "one_key":
        q = np.full(nq, keys[7], dtype=np.uint64)
    elif pattern == "two_keys":
        q = np.where(np.arange(nq) % 2 == 0, keys[1], keys[2]).astype(np.uint64)
    else:
        q = np.concatenate([keys] * 15 + [keys[:nq - 15 * n]])
        q = np.sort(q)  # clusters equal keys, and runs of tiles share groups unevenly
    d_q = torch.from_numpy(q.view(np.int64)).cuda()
    for minimal in (True, False):
        want = ri.query_u64(q, minimal, "loop", threads=THREADS)
        out = idx.query(d_q, minimal=minimal, out_width=8)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy().view(np.uint64), want), minimal


@pytest.mark.parametrize("koff,ooff", [(1, 0), (0, 1), (1, 3), (2, 2)])
def test_partitioned_unaligned_buffers(ph, ref, koff, ooff):
    """Keys / outputs not 16-B aligned take the register-staged kernels instead of the
    bulk-copy ones (pass A needs aligned keys, pass C's bulk store an aligned output)."""
    from oracle.bindings import corpus_u64_np
    n = 150_000
    keys = corpus_u64_np(0, n, 64)
    ptrh = ref.build_u64(keys, ref.params("default", lambda_=(30, 10)))
    ri = ref.load(ptrh)
    idx = ph.PtrHashIndex(ptrh)
    nq = 2 * (1 << 20) + 5
    q = corpus_u64_np(0, nq, 65)
    q[:n] = keys
    want = ri.query_u64(q, True, "loop", threads=THREADS)
    base = torch.zeros(nq + koff, dtype=torch.int64, device="cuda")
    base[koff:] = torch.from_numpy(q.view(np.int64)).cuda()
    obuf = torch.zeros(nq + ooff, dtype=torch.int32, device="cuda")
    out = obuf[ooff:]
    idx.query(base[koff:], out=out, minimal=True, out_width=4)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy().view(np.uint32).astype(np.uint64), want)


@pytest.mark.parametrize("slice_kb,nq", [(40, 1_000_003), (24, 2 * (1 << 20) + 11), (12, 1_000_003)])
def test_partitioned_many_groups(ph, ref, slice_kb, nq, monkeypatch):
    """Small pilot slices force many groups: ~17 and ~28 (bulk-copy pass A, lane = group)
    and ~56 (> 32: the register-staged pass A)."""
    from oracle.bindings import corpus_u64_np
    n = 2_000_000
    keys = corpus_u64_np(0, n, 66)
    ptrh = ref.build_u64(keys, ref.params("default", lambda_=(30, 10)))
    ri = ref.load(ptrh)
    idx = ph.PtrHashIndex(ptrh)
    q = corpus_u64_np(0, nq, 67)
    q[: min(nq, n) // 2] = keys[: min(nq, n) // 2]
    d_q = torch.from_numpy(q.view(np.int64)).cuda()
    monkeypatch.setenv("PH_GPU_PART_SLICE_KB", str(slice_kb))
    for minimal in (True, False):
        want = ri.query_u64(q, minimal, "loop", threads=THREADS)
        out = idx.query(d_q, minimal=minimal, out_width=4)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy().view(np.uint32).astype(np.uint64), want), minimal


def test_trim_releases_scratch_between_calls(ph, ref):
    """ph_gpu_index_trim after a partitioned call: later calls allocate again and agree."""
    from oracle.bindings import corpus_u64_np
    n = 200_000
    keys = corpus_u64_np(0, n, 71)
    ptrh = ref.build_u64(keys, ref.params("default", lambda_=(30, 10)))
    idx = ph.PtrHashIndex(ptrh)
    d_q = torch.from_numpy(keys.view(np.int64)).cuda()
    a = idx.query(d_q, minimal=True, out_width=4)
    torch.cuda.synchronize()
    idx.trim()
    b = idx.query(d_q, minimal=True, out_width=4)
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    assert np.array_equal(np.sort(b.cpu().numpy().view(np.uint32)), np.arange(n, dtype=np.uint32))


def test_pass_timing_records_three_passes(ph, ref):
    """ph_gpu_set_pass_timing / ph_gpu_pass_times: one partitioned call records positive
    times for the bin, query and unbin passes; direct-path calls record nothing."""
    from oracle.bindings import corpus_u64_np
    n = 300_000
    keys = corpus_u64_np(0, n, 68)
    idx = ph.PtrHashIndex(ref.build_u64(keys, ref.params("default", lambda_=(30, 10))))
    d_q = torch.from_numpy(keys.view(np.int64)).cuda()
    ph.set_pass_timing(True)
    try:
        idx.query(d_q, minimal=True, out_width=4)
        ms, calls = ph.pass_times()
        assert calls == 1 and all(t > 0 for t in ms), (ms, calls)
        ph.set_partition(1)  # direct kernel: no pass events
        idx.query(d_q, minimal=True, out_width=4)
        ph.set_partition(2)
        assert ph.pass_times()[1] == 1
    finally:
        ph.set_pass_timing(False)


@pytest.mark.parametrize("n_bases,k,woff", [(100, 31, 0), (4096 + 30, 31, 0), (130 * 32 + 31, 31, 0),
                                            (300_017, 31, 1), (300_017, 16, 0), (250_000, 32, 1),
                                            (200_003, 9, 0)])
def test_partitioned_kmers_edges(ph, ref, port, n_bases, k, woff):
    """Partitioned k-mer path: partial and single tiles, the last tiles whose 130 packed
    words run past the sequence (loaded without the bulk engine), other k, and a sequence
    that is only 8-B aligned (woff = 1: no bulk loads at all)."""
    seq = port.gen_dna(n_bases, 46 + k)
    kmers = port.kmers(seq, n_bases, k)
    uniq = np.unique(kmers)
    ptrh = ref.build_u64(uniq, ref.params("default", lambda_=(30, 10)))
    ri = ref.load(ptrh)
    idx = ph.PtrHashIndex(ptrh)
    buf = torch.zeros(seq.size + woff, dtype=torch.int64, device="cuda")
    buf[woff:] = torch.from_numpy(seq.view(np.int64)).cuda()
    for minimal in (True, False):
        want = ri.query_u64(kmers, minimal, "loop", threads=THREADS)
        out = idx.query_kmers(buf[woff:], n_bases, k, minimal=minimal, out_width=8)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy().view(np.uint64), want), (n_bases, k, woff, minimal)


def test_partitioned_concurrent_streams(ph, ref):
    """Several host threads query one index through the partitioned path on their own
    streams at once (per-call scratch from the index's stream-ordered pool): every output
    equals the reference's."""
    import threading
    from oracle.bindings import corpus_u64_np
    n = 250_000
    keys = corpus_u64_np(0, n, 69)
    ptrh = ref.build_u64(keys, ref.params("default", lambda_=(30, 10)))
    ri = ref.load(ptrh)
    idx = ph.PtrHashIndex(ptrh)
    qs = [corpus_u64_np(0, 1_500_000 + 4097 * t, 70 + t) for t in range(4)]
    for q in qs:
        q[:n] = keys
    wants = [ri.query_u64(q, True, "loop", threads=THREADS) for q in qs]
    outs = [None] * len(qs)
    errs = []

    def work(t):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                d = torch.from_numpy(qs[t].view(np.int64)).cuda()
                for _ in range(3):
                    o = idx.query(d, minimal=True, out_width=4, stream=s.cuda_stream)
                s.synchronize()
                outs[t] = o.cpu().numpy().view(np.uint32).astype(np.uint64)
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=work, args=(t,)) for t in range(len(qs))]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert not errs, errs
    for t in range(len(qs)):
        assert np.array_equal(outs[t], wants[t]), t


def test_auto_partition_on_dram_sized_index(ref):
    """Default settings end to end: an index whose pilot array exceeds 64 MiB keeps the file
    order without a window, and a device batch above pilot_bytes/32 takes the partitioned
    path by itself (the pass timers see it). Every key checked against the reference on a
    sample and the minimal outputs a bijection on all of them."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from oracle.bindings import corpus_u64_np
    from paper_2502_15539_b200 import ph_gpu
    n = 220_000_000
    keys = corpus_u64_np(0, n, 84)
    ptrh = ref.build_u64(keys, ref.params("default", lambda_=(30, 10)))
    idx = ph_gpu.PtrHashIndex(ptrh)
    assert idx.info.pilot_bytes > (64 << 20)
    ph_gpu.set_partition(0)
    d_k = torch.from_numpy(keys.view(np.int64)).cuda()
    ph_gpu.set_pass_timing(True)
    try:
        out = idx.query(d_k, minimal=True, out_width=4)
        torch.cuda.synchronize()
        assert ph_gpu.pass_times()[1] == 1  # the partitioned path ran
    finally:
        ph_gpu.set_pass_timing(False)
    oob, dups = idx.verify_bijection(out)
    assert oob == 0 and dups == 0
    ri = ref.load(ptrh)
    rng = np.random.default_rng(5)
    sample = np.sort(rng.choice(n, 2_000_000, replace=False))
    want = ri.query_u64(keys[sample], True, "loop", threads=THREADS)
    got = out.cpu().numpy().view(np.uint32)[sample].astype(np.uint64)
    assert np.array_equal(got, want)
