"""GPU tests of the two remap paths: the inline warp-compacted decode
(batches < 2^20 keys) and the deferred list + k_remap_patch (larger batches), including
list overflow (remap fraction far above the list's n/32 capacity), against the reference."""
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
    return ph_gpu


@pytest.mark.parametrize("alpha,remap", [((99, 100), "cacheline-ef"), ((90, 100), "cacheline-ef"),
                                         ((80, 100), "plain32"), ((90, 100), "elias-fano")])
@pytest.mark.parametrize("nq", [(1 << 20) - 1, (1 << 20) + 12345, 3_000_000])
def test_deferred_and_inline_remap(ph, ref, alpha, remap, nq):
    from oracle.bindings import corpus_u64_np
    n = 400_000
    keys = corpus_u64_np(0, n, 51)
    ptrh = ref.build_u64(keys, ref.params("default", lambda_=(30, 10), alpha=alpha, remap=remap))
    ri = ref.load(ptrh)
    idx = ph.PtrHashIndex(ptrh)
    q = corpus_u64_np(0, nq, 52)  # mostly non-members: remap rate ~ 1 - alpha
    q[: n // 2] = keys[: n // 2]
    want = ri.query_u64(q, True, "loop", threads=THREADS)
    d_q = torch.from_numpy(q.view(np.int64)).cuda()
    for width in (4, 8):
        out = idx.query(d_q, minimal=True, out_width=width)
        torch.cuda.synchronize()
        got = out.cpu().numpy().view(np.uint32 if width == 4 else np.uint64).astype(np.uint64)
        assert np.array_equal(got, want)
    assert np.array_equal(idx.query(q, minimal=True, out_width=4).astype(np.uint64), want)
