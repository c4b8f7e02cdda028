"""Construction assist: the front phases of one u64 build attempt —
hash_all, scatter_to_parts, per-part sort + duplicate check (construction.cpp:98-111,
engine.hpp:412-518). CPU: the numpy restatement equals the reference's own code; GPU:
ph_gpu_build_prepare_u64 equals the reference bit for bit."""
import numpy as np
import pytest

from oracle.bindings import build_prepare_u64_np, corpus_u64_np


def _cases(ref):
    keys = corpus_u64_np(0, 300_000, 81)
    P, S, _ = ref.shape(keys.size, ref.params("default", lambda_=(30, 10)))
    seed = 0x9E3779B97F4A7C15
    dup = keys.copy()
    dup[-1] = dup[5]  # two equal keys: equal hashes
    return [("ok", keys, P, S, seed, 0), ("dup", dup, P, S, seed, 2),
            ("oversubscribed", keys, P, (keys.size // P) // 2, seed, 1),
            ("one_part", keys[:5000], 1, 6000, 12345, 0), ("empty_parts", keys[:50], 64, 10, seed, 0)]


def test_numpy_restatement_matches_reference(ref):
    for name, keys, P, S, seed, want in _cases(ref):
        h_r, off_r, st_r = ref.build_prepare_u64(keys, P, S, seed)
        h_n, off_n, st_n = build_prepare_u64_np(keys, P, S, seed)
        assert st_r == st_n == want, name
        if st_r != 1:  # on kOversubscribed the reference stops before sorting
            assert np.array_equal(h_r, h_n), name
            assert np.array_equal(off_r, off_n), name


@pytest.mark.gpu
def test_gpu_build_prepare_matches_reference(ref):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2502_15539_b200 import ph_gpu
    for name, keys, P, S, seed, want in _cases(ref):
        h_r, off_r, st_r = ref.build_prepare_u64(keys, P, S, seed)
        d_k = torch.from_numpy(keys.view(np.int64)).cuda()
        before = ph_gpu.launch_count()
        h, off, st = ph_gpu.build_prepare_u64(d_k, P, S, seed)
        assert ph_gpu.launch_count() > before
        assert st == st_r == want, name
        if st != 1:
            assert np.array_equal(h.cpu().numpy().view(np.uint64), h_r), name
            assert np.array_equal(off.cpu().numpy().view(np.uint64), off_r), name


@pytest.mark.gpu
@pytest.mark.parametrize("preset,fn", [("default", None), ("fast", None), ("default", "quadratic"),
                                       ("default", "skewed"), ("default", "optimal")])
def test_gpu_bucket_sizes_match_reference_stats(ref, preset, fn):
    """ph_gpu_bucket_sizes over the build's key set equals the reference's
    BuildStats::bucket_size_counts (stats.cpp:59-61) for every bucket function."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2502_15539_b200 import ph_gpu
    keys = corpus_u64_np(0, 400_000, 82)
    params = ref.params(preset, lambda_=(30, 10)) if fn is None else \
        ref.params(preset, lambda_=(30, 10), bucket_fn=fn)
    ptrh, want = ref.build_u64_stats(keys, params)
    idx = ph_gpu.PtrHashIndex(ptrh)
    got = idx.bucket_sizes(torch.from_numpy(keys.view(np.int64)).cuda())
    assert np.array_equal(got, want), (preset, fn)


@pytest.mark.gpu
@pytest.mark.parametrize("n", [0, 1, 2, 4097])
def test_gpu_build_prepare_tiny(n):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2502_15539_b200 import ph_gpu
    keys = corpus_u64_np(0, n, 83)
    P, S, seed = 7, 1000, 12345
    h_n, off_n, st_n = build_prepare_u64_np(keys, P, S, seed)
    h, off, st = ph_gpu.build_prepare_u64(torch.from_numpy(keys.view(np.int64)).cuda(), P, S, seed)
    assert st == st_n
    assert np.array_equal(h.cpu().numpy().view(np.uint64), h_n)
    assert np.array_equal(off.cpu().numpy().view(np.uint64), off_n)
