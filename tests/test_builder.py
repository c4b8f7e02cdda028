"""Construction: ph_gpu_build_u64 / ph_build_from_sorted_u64 produce the same
PTRH bytes as the reference's build() + serialize() (construction.cpp:139-152,
serde.cpp:142-170) for the same keys and parameters.

CPU: the host stage (per-part pilot search, remap assembly, serialization; engine.hpp:105-557)
fed with the numpy restatement of the front phases, against the reference's own build, for
every bucket function, remap kind and reduce kind, forced shapes and the error paths
(mirrors test_construction.cpp and test_shape.cpp). GPU: the whole build, with the front on
the device (hand-written sort, ph_sort.cu), host- and device-resident keys, reseeding,
duplicate keys, and skewed hash sets that exercise every split level of the sort."""
import numpy as np
import pytest

from oracle.bindings import build_prepare_u64_np, corpus_u64_np

CASES = [
    ("default", dict(lambda_=(30, 10))),
    ("default", {}),
    ("fast", {}),
    ("compact", {}),
    ("default", dict(bucket_fn="linear", lambda_=(30, 10))),
    ("default", dict(bucket_fn="quadratic")),
    ("default", dict(bucket_fn="skewed", remap="elias-fano")),
    ("default", dict(bucket_fn="optimal", remap="plain32")),
    ("compact", dict(reduce="pow2-mul")),
    ("fast", dict(reduce="pow2-mul", remap="elias-fano")),
    ("default", dict(reduce="fastmod-single")),
    ("default", dict(alpha=(98, 100), lambda_=(42, 10))),
]


def _ph():
    from paper_2502_15539_b200 import ph_gpu
    return ph_gpu


def _seed_of(ptrh: bytes) -> int:
    return int.from_bytes(ptrh[48:56], "little")


def _host_build(ph, keys, gp, threads=0):
    """The attempt loop of build_u64_impl (construction.cpp:113-138) with the numpy front."""
    P, S, _ = (gp.parts, gp.slots_per_part, gp.buckets_per_part) if gp.parts else \
        ph.compute_shape(keys.size, gp)
    seed = gp.seed
    for attempt in range(gp.max_seed_retries + 1):
        h, off, st = build_prepare_u64_np(keys, P, S, seed)
        if st == 2:
            raise ph.PhGpuError(ph.E_DUPLICATE, "duplicate keys")
        if st == 0:
            try:
                return ph.build_from_sorted_u64(h, off, gp, seed, threads=threads)
            except ph.PhGpuError as e:
                if e.code != ph.E_BUILD_FAILED:
                    raise
        seed = (0x517CC1B727220A95 * ((seed ^ attempt) ^ 0x9E3779B97F4A7C15)) & ((1 << 64) - 1)
    raise ph.PhGpuError(ph.E_BUILD_FAILED, "all attempts failed")


@pytest.mark.parametrize("preset,kw", CASES)
def test_host_stage_matches_reference(ref, preset, kw):
    ph = _ph()
    keys = corpus_u64_np(0, 150_000, 91)
    want = ref.build_u64(keys, ref.params(preset, **kw))
    gp = ph.build_params(preset, **kw)
    assert ph.compute_shape(keys.size, gp) == ref.shape(keys.size, ref.params(preset, **kw))
    got = _host_build(ph, keys, gp, threads=4)
    assert got == want, (preset, kw)


@pytest.mark.parametrize("n", [1, 2, 3, 45, 1000, 44 * 37])
def test_host_stage_tiny(ref, n):
    ph = _ph()
    keys = corpus_u64_np(0, n, 92)
    for preset in ("default", "fast"):
        assert _host_build(ph, keys, ph.build_params(preset)) == ref.build_u64(keys, ref.params(preset)), (n, preset)


@pytest.mark.parametrize("shape", [(1, 6000, 1700), (7, 800, 250), (16, 1 << 9, 180), (3, 1877, 2000)])
def test_host_stage_forced_shape(ref, shape):
    """build_with_shape (construction.cpp:145-152), including tight shapes that need reseeds."""
    ph = _ph()
    keys = corpus_u64_np(0, 5000, 93)
    P, S, B = shape
    want = ref.build_u64_shape(keys, ref.params("default", lambda_=(30, 10)), P, S, B)
    got = _host_build(ph, keys, ph.build_params("default", lambda_=(30, 10), shape=shape))
    assert got == want, shape


def test_reseed_path_matches_reference(ref):
    """A shape tight enough that the first seeds fail (oversubscribed parts or failed
    placement): the accepted seed and the bytes equal the reference's."""
    ph = _ph()
    keys = corpus_u64_np(0, 4000, 94)
    shape = (8, 520, 170)  # 4160 slots for 4000 keys: the default seed fails
    rp = ref.params("fast", retries=30)
    want = ref.build_u64_shape(keys, rp, *shape)
    got = _host_build(ph, keys, ph.build_params("fast", retries=30, shape=shape))
    assert got == want
    assert _seed_of(want) != rp.seed  # the case really reseeded


def test_hopeless_shape_fails_like_reference(ref):
    ph = _ph()
    keys = corpus_u64_np(0, 4000, 94)
    with pytest.raises(RuntimeError):
        ref.build_u64_shape(keys, ref.params("fast", retries=2, alpha=(1, 1)), 1, 4000, 1)
    with pytest.raises(ph.PhGpuError) as e:
        _host_build(ph, keys, ph.build_params("fast", retries=2, shape=(1, 4000, 1), alpha=(1, 1)))
    assert e.value.code == ph.E_BUILD_FAILED


def test_compute_shape_matches_reference(ref):
    ph = _ph()
    for n in [1, 2, 100, 79_999, 80_000, 80_001, 10**6, 10**7, 10**8, 10**9, 3 * 10**8, 2**32 - 1]:
        for preset, kw in CASES:
            try:
                want = ref.shape(n, ref.params(preset, **kw))
            except ValueError:
                with pytest.raises(ph.PhGpuError):
                    ph.compute_shape(n, ph.build_params(preset, **kw))
                continue
            assert ph.compute_shape(n, ph.build_params(preset, **kw)) == want, (n, preset, kw)


def test_invalid_params_rejected():
    ph = _ph()
    keys = corpus_u64_np(0, 100, 95)
    h, off, _ = build_prepare_u64_np(keys, 1, 200, 1)
    bad = [dict(alpha=(0, 100)), dict(alpha=(101, 100)), dict(lambda_=(9, 10)),
           dict(alpha=(995, 1000))]  # CacheLineEF needs alpha <= 0.99 (shape.cpp:58-62)
    for kw in bad:
        with pytest.raises(ph.PhGpuError) as e:
            ph.build_from_sorted_u64(h, off, ph.build_params("default", **kw), 1)
        assert e.value.code == ph.E_INVALID, kw
    with pytest.raises(ph.PhGpuError) as e:
        ph.build_params("nope")
    assert e.value.code == ph.E_INVALID
    with pytest.raises(ph.PhGpuError) as e:  # fewer slots than keys
        ph.build_from_sorted_u64(h, off, ph.build_params("default", shape=(1, 50, 20)), 1)
    assert e.value.code == ph.E_INVALID


# ---- GPU: the whole build ----

def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.fixture(params=[1, 2], ids=["host_search", "gpu_search"])
def search_mode(request):
    """Both homes of the pilot search: host threads (1) and the GPU kernel (2, no fallback)."""
    ph = _ph()
    ph.set_build_search(request.param)
    yield request.param
    ph.set_build_search(0)


@pytest.mark.gpu
@pytest.mark.parametrize("preset,kw", CASES)
def test_gpu_build_matches_reference(ref, preset, kw, search_mode):
    torch = _cuda()
    ph = _ph()
    keys = corpus_u64_np(0, 300_000, 96)
    want = ref.build_u64(keys, ref.params(preset, **kw))
    before = ph.launch_count()
    got, st = ph.build_u64(keys, ph.build_params(preset, **kw), stats=True)
    assert ph.launch_count() > before  # the front ran on the device
    assert got == want, (preset, kw)
    assert st["n"] == keys.size and st["attempts"] >= 1
    assert st["search_on_gpu"] == (search_mode == 2)
    # device-resident keys give the same bytes
    d = torch.from_numpy(keys.view(np.int64)).cuda()
    assert ph.build_u64(d, ph.build_params(preset, **kw)) == want


@pytest.mark.gpu
def test_gpu_search_stats_match_host_search(ref):
    """Evictions (total and by percentile of first placements) are a trace of the search's
    order and choices: the GPU search reports the host search's numbers exactly."""
    _cuda()
    ph = _ph()
    keys = corpus_u64_np(0, 2_000_000, 91)
    bp = ph.build_params("compact")  # lambda 4.0: evictions in every part
    try:
        ph.set_build_search(1)
        b1, s1 = ph.build_u64(keys, bp, stats=True)
        ph.set_build_search(2)
        b2, s2 = ph.build_u64(keys, bp, stats=True)
    finally:
        ph.set_build_search(0)
    assert b1 == b2 == ref.build_u64(keys, ref.params("compact"))
    assert s2["search_on_gpu"] and not s1["search_on_gpu"]
    assert s1["total_evictions"] == s2["total_evictions"] > 0
    assert s1["evictions_by_percentile"] == s2["evictions_by_percentile"]


@pytest.mark.gpu
def test_gpu_build_reseed_and_errors(ref, search_mode):
    _cuda()
    ph = _ph()
    keys = corpus_u64_np(0, 4000, 94)
    shape = (8, 520, 170)
    want = ref.build_u64_shape(keys, ref.params("fast", retries=30), *shape)
    assert ph.build_u64(keys, ph.build_params("fast", retries=30, shape=shape)) == want
    dup = corpus_u64_np(0, 50_000, 97)
    dup[-1] = dup[17]
    with pytest.raises(ph.PhGpuError) as e:
        ph.build_u64(dup)
    assert e.value.code == ph.E_DUPLICATE
    with pytest.raises(ph.PhGpuError) as e:  # one bucket of 4000 keys: no pilot is collision-free
        ph.build_u64(keys, ph.build_params("fast", retries=2, shape=(1, 4000, 1), alpha=(1, 1)))
    assert e.value.code == ph.E_BUILD_FAILED  # in either home of the search
    with pytest.raises(ph.PhGpuError) as e:
        ph.build_u64(keys[:0])
    assert e.value.code == ph.E_INVALID


@pytest.mark.gpu
def test_gpu_build_large_matches_reference(ref, search_mode):
    """n = 2e7: 16 parts of ~1.2 M keys, two split levels in the device sort, the pinned
    transfer ring in several chunks; byte-identical to the reference's build."""
    _cuda()
    ph = _ph()
    keys = corpus_u64_np(0, 20_000_000, 42)
    rp = ref.params("default", lambda_=(30, 10))
    want = ref.build_u64(keys, rp)
    got, st = ph.build_u64(keys, ph.build_params("default", lambda_=(30, 10)), stats=True)
    assert got == want
    assert st["prepare_ms"] > 0 and st["search_ms"] > 0


def _keys_for_hashes(ref, h: np.ndarray, seed: int) -> np.ndarray:
    """Keys whose hashes C*(key^seed) are exactly h (C is odd, so invertible mod 2^64)."""
    cinv = np.uint64(ref.L.ref_mix_constant_inverse())
    with np.errstate(over="ignore"):
        return (h.astype(np.uint64) * cinv) ^ np.uint64(seed)


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["narrow", "clustered", "repeated", "uniform_big"])
def test_gpu_sort_skewed_hash_sets(ref, kind):
    """The device MSD sort on hash sets that defeat its fast path: all hashes in a 2^20
    window (every split level and the redo path down to the last 12 bits), clusters of
    equal high bits with bins over 64 keys, many repeated values (duplicates), and a
    uniform set large enough for two split levels. Compared with numpy's sort."""
    torch = _cuda()
    ph = _ph()
    rng = np.random.default_rng(7)
    seed = 0x9E3779B97F4A7C15
    if kind == "narrow":
        h = np.uint64(0xABCDE) << np.uint64(40) | rng.integers(0, 1 << 20, 300_000, dtype=np.uint64)
    elif kind == "clustered":
        hi = rng.integers(0, 64, 400_000, dtype=np.uint64) << np.uint64(50)
        h = hi | (rng.integers(0, 1 << 10, 400_000, dtype=np.uint64) << np.uint64(20)) | \
            rng.integers(0, 1 << 20, 400_000, dtype=np.uint64)
    elif kind == "repeated":
        h = rng.integers(0, 1000, 200_000, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15)
    else:
        h = rng.integers(0, 2**63, 30_000_000, dtype=np.uint64) * np.uint64(2) + np.uint64(1)
    keys = _keys_for_hashes(ref, h, seed)
    P, S = 5, 10**9
    want_h, want_off, want_st = build_prepare_u64_np(keys, P, S, seed)
    got_h, got_off, st = ph.build_prepare_u64(torch.from_numpy(keys.view(np.int64)).cuda(), P, S, seed)
    assert st == want_st
    assert np.array_equal(got_h.cpu().numpy().view(np.uint64), want_h), kind
    assert np.array_equal(got_off.cpu().numpy().view(np.uint64), want_off), kind

@pytest.mark.gpu
def test_gpu_search_random_shapes_match_host_search():
    """Seeded sweep over key counts, lambda, alpha, bucket functions, reduce kinds and forced
    shapes (tiny S: the 64-bit mod; pow2 S; few buckets: big buckets and big-bucket evictions;
    tight shapes: many evictions, reseeds and failures): the GPU search and the host search give
    the same bytes or fail with the same code."""
    _cuda()
    ph = _ph()
    rng = np.random.default_rng(20260)
    fns = ["linear", "quadratic", "cubic", "skewed", "optimal"]
    ran = unsupported = failed = 0
    try:
        for case in range(30):
            n = int(rng.choice([700, 5_000, 40_000, 150_000]))
            keys = corpus_u64_np(0, n, 500 + case)
            kw = dict(bucket_fn=str(rng.choice(fns)), lambda_=(int(rng.integers(12, 60)), 10),
                      alpha=(int(rng.integers(90, 100)), 100), retries=1,
                      reduce=str(rng.choice(["fastmod-multi", "pow2-mul"])),
                      remap=str(rng.choice(["plain32", "elias-fano"])))
            if case % 3 == 0:  # a forced shape: P parts, S slots, B buckets
                P = int(rng.choice([1, 3, 7]))
                S = int(n / P * rng.uniform(1.02, 1.3)) + 8
                if kw["reduce"] == "pow2-mul":
                    S = 1 << int(np.ceil(np.log2(S)))
                B = max(1, int(n / P / rng.uniform(1.5, 40.0)))
                kw["shape"] = (P, S, B)
            res = []
            for mode in (1, 2):
                ph.set_build_search(mode)
                try:
                    res.append(("ok", ph.build_u64(keys, ph.build_params("default", **kw))))
                except ph.PhGpuError as e:
                    res.append(("err", e.code))
            if res[1] == ("err", ph.E_UNSUPPORTED):
                unsupported += 1
                continue
            assert res[0] == res[1], (case, n, kw, res[0][0], res[1][0])
            ran += 1
            failed += res[0][0] == "err"
    finally:
        ph.set_build_search(0)
    assert ran >= 20 and ran - failed >= 12, (ran, failed, unsupported)

@pytest.mark.gpu
def test_gpu_search_falls_back_for_large_parts(ref):
    """A part whose occupancy bitmap does not fit one CTA's shared memory (S = 2e6 slots) is
    searched on host threads in the default mode (same bytes as the reference) and refused
    with E_UNSUPPORTED when the GPU search is forced."""
    _cuda()
    ph = _ph()
    keys = corpus_u64_np(0, 60_000, 77)
    shape = (1, 2_000_000, 20_000)
    want = ref.build_u64_shape(keys, ref.params("default", lambda_=(30, 10)), *shape)
    got, st = ph.build_u64(keys, ph.build_params("default", lambda_=(30, 10), shape=shape), stats=True)
    assert got == want and not st["search_on_gpu"]
    ph.set_build_search(2)
    try:
        with pytest.raises(ph.PhGpuError) as e:
            ph.build_u64(keys, ph.build_params("default", lambda_=(30, 10), shape=shape))
        assert e.value.code == ph.E_UNSUPPORTED
        # S = 1.2e6: the bitmap fits one CTA per SM (not two): still the GPU search, same bytes
        shape1 = (1, 1_200_000, 20_000)
        want1 = ref.build_u64_shape(keys, ref.params("default", lambda_=(30, 10)), *shape1)
        got1, st1 = ph.build_u64(keys, ph.build_params("default", lambda_=(30, 10), shape=shape1), stats=True)
        assert got1 == want1 and st1["search_on_gpu"]
    finally:
        ph.set_build_search(0)

# ---- GPU: string-key builds ----

def _concat(strs):
    offs = np.zeros(len(strs) + 1, dtype=np.uint64)
    offs[1:] = np.cumsum([len(s) for s in strs])
    data = np.frombuffer(b"".join(strs) or b"\0", dtype=np.uint8).copy()
    return data, offs


@pytest.mark.gpu
@pytest.mark.parametrize("preset,kw", [("default", dict(lambda_=(30, 10))), ("fast", {}),
                                       ("compact", dict(remap="elias-fano"))])
def test_gpu_build_bytes_matches_reference(ref, preset, kw, search_mode):
    """build(span<const std::string>) + serialize(): the string hash (aes64, what the reference
    picks on this host) runs on the GPU and the 64-bit hashes go through the u64 front and the
    pilot search; the bytes equal the reference's, from host and from device buffers, with the
    edge lengths (empty, 1, 15, 16, 17, 200, 1024 bytes) among the keys."""
    torch = _cuda()
    ph = _ph()
    from oracle.bindings import string_corpus
    strs = string_corpus(120_000, 31) + [b"", b"a", b"q" * 15, b"x" * 16, b"y" * 17, b"z" * 200,
                                         bytes(range(256)) * 4]
    data, offs = _concat(strs)
    want = ref.build_bytes(data, offs, ref.params(preset, **kw))
    assert want[8] == 1 and want[9] == 1, "the reference picked another string hash on this host"
    got, st = ph.build_bytes(data, offs, ph.build_params(preset, **kw), hash_algo=1, stats=True)
    assert got == want
    assert st["n"] == len(strs) and st["search_on_gpu"] == (search_mode == 2)
    d = torch.from_numpy(data).cuda()
    o = torch.from_numpy(offs.view(np.int64)).cuda()
    assert ph.build_bytes(d, o, ph.build_params(preset, **kw), hash_algo=1) == want


@pytest.mark.gpu
def test_gpu_build_bytes_portable64_and_errors(ref):
    """portable64 (the reference's choice on hosts without AES-NI): the built index is a
    bijection on its keys when queried through the GPU path, and identical keys (equal
    fingerprints under every seed) end like the reference's persistent-duplicate failure."""
    _cuda()
    ph = _ph()
    from oracle.bindings import string_corpus
    strs = string_corpus(60_000, 32)
    data, offs = _concat(strs)
    b = ph.build_bytes(data, offs, ph.build_params("default", lambda_=(30, 10)), hash_algo=3)
    assert b[8] == 1 and b[9] == 3
    idx = ph.PtrHashIndex(b)
    got = idx.query((data, offs), out_width=4).astype(np.uint64)
    assert np.array_equal(np.sort(got), np.arange(len(strs), dtype=np.uint64))
    dup = strs[:1000] + [strs[7]]
    d2, o2 = _concat(dup)
    with pytest.raises(ph.PhGpuError) as e:
        ph.build_bytes(d2, o2, ph.build_params("default"), hash_algo=1)
    assert e.value.code == ph.E_UNSUPPORTED
    with pytest.raises(ph.PhGpuError) as e:
        ph.build_bytes(data, offs, ph.build_params("default"), hash_algo=2)
    assert e.value.code == ph.E_UNSUPPORTED

@pytest.mark.gpu
def test_gpu_build_tiny_inputs(ref):
    """1 to 1000 keys (parts with a single bucket, a single key, the empty string as a key):
    u64 and string builds with the GPU search forced give the reference's bytes."""
    _cuda()
    ph = _ph()
    from oracle.bindings import string_corpus
    ph.set_build_search(2)
    try:
        for n in (1, 2, 3, 7, 33, 257, 1000):
            keys = corpus_u64_np(0, n, 1000 + n)
            for preset in ("default", "fast", "compact"):
                got, st = ph.build_u64(keys, ph.build_params(preset), stats=True)
                assert got == ref.build_u64(keys, ref.params(preset)) and st["search_on_gpu"], (n, preset)
            strs = string_corpus(n, n, 0, 40) if n > 1 else [b""]
            data, offs = _concat(strs)
            assert ph.build_bytes(data, offs, ph.build_params("default")) == \
                ref.build_bytes(data, offs, ref.params("default")), ("strings", n)
    finally:
        ph.set_build_search(0)
