"""Host-API behaviour of the C ABI on the GPU: single-key latency (no allocation per call),
the shared persisting-L2 set-aside across indexes, residency checks of the host-span entry
points, and the Python wrapper's argument checks with device tensors."""
import ctypes as C
import os
import statistics
import sys
import time

import numpy as np
import pytest

from conftest import ROOT

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ph():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2502_15539_b200 import ph_gpu
    return ph_gpu


def _persisting_limit():
    from cuda.bindings import runtime as rt  # cuda-python; same primary context
    err, v = rt.cudaDeviceGetLimit(rt.cudaLimit.cudaLimitPersistingL2CacheSize)
    assert err == rt.cudaError_t.cudaSuccess
    return int(v)


def test_single_key_latency_u64(ph, ref):
    """index(key) is a drop-in for the reference's single-key call (index.hpp:60-64): no
    device allocation or copy call per key; median latency <= 20 us on a B200."""
    from oracle.bindings import corpus_u64_np
    n = 100_000
    keys = corpus_u64_np(0, n, 5)
    ptrh = ref.build_u64(keys, ref.params("default", lambda_=(30, 10)))
    ri = ref.load(ptrh)
    idx = ph.PtrHashIndex(ptrh)
    q = np.concatenate([keys[:500], corpus_u64_np(0, 500, 6)])
    for k in q[:50]:
        idx.index(int(k))
    ts = []
    for k in q:
        t = time.perf_counter()
        got = idx.index(int(k))
        ts.append(time.perf_counter() - t)
        assert got == ri.index(int(k), True)
    for k in q[:100]:
        assert idx.index_no_remap(int(k)) == ri.index(int(k), False)
    med = statistics.median(ts) * 1e6
    print(f"single-key u64 latency: median {med:.1f} us, p90 {sorted(ts)[len(ts) * 9 // 10] * 1e6:.1f} us")
    assert med <= 20.0


def test_single_key_latency_bytes(ph, ref):
    from oracle.bindings import string_corpus
    strs = string_corpus(20_000, 9)
    data = np.frombuffer(b"".join(strs), dtype=np.uint8)
    offs = np.zeros(len(strs) + 1, dtype=np.uint64)
    offs[1:] = np.cumsum([len(s) for s in strs])
    ptrh = ref.build_bytes(data, offs, ref.params("default", lambda_=(30, 10)))
    ri = ref.load(ptrh)
    idx = ph.PtrHashIndex(ptrh)
    ts = []
    long_key = b"x" * 5000  # grows the scratch block once
    for s in strs[:300] + [long_key, b""]:
        t = time.perf_counter()
        got = idx.index(s)
        ts.append(time.perf_counter() - t)
        one = np.frombuffer(s or b"\0", dtype=np.uint8)
        want = ri.query_bytes(one, np.array([0, len(s)], dtype=np.uint64), True, "single")[0]
        assert got == want
    med = statistics.median(ts) * 1e6
    print(f"single-key string latency: median {med:.1f} us")
    assert med <= 20.0


def test_small_window_survives_large_index(ph, ref):
    """A DRAM-sized index created after a small windowed one must not cancel the small one's
    persisting set-aside; the set-aside goes when the last window owner goes."""
    from oracle.bindings import corpus_u64_np
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    from synth_perf import synth_ptrh
    keys = corpus_u64_np(0, 200_000, 3)
    small_ptrh = ref.build_u64(keys, ref.params("default", lambda_=(30, 10)))
    ri = ref.load(small_ptrh)
    small = ph.PtrHashIndex(small_ptrh)
    lim_small = _persisting_limit()
    assert lim_small > 0, "a small index keeps its pilots under a persisting window"
    large = ph.PtrHashIndex(synth_ptrh(4))  # 100 MB of pilots: no window of its own
    assert large.info.pilot_bytes > (64 << 20)
    assert _persisting_limit() >= lim_small
    got = small.query(torch.from_numpy(keys.view(np.int64)).cuda(), minimal=True, out_width=8)
    torch.cuda.synchronize()
    assert np.array_equal(got.cpu().numpy().view(np.uint64), ri.query_u64(keys, True, "loop"))
    small.close()
    assert _persisting_limit() == 0, "no live window: the set-aside is released"
    large.close()


def test_stream_entry_points_reject_mixed_residency(ph, ref):
    from oracle.bindings import corpus_u64_np
    keys = corpus_u64_np(0, 50_000, 4)
    idx = ph.PtrHashIndex(ref.build_u64(keys, ref.params("default", lambda_=(30, 10))))
    d_keys = torch.from_numpy(keys.view(np.int64)).cuda()
    h_out = np.zeros(keys.size, dtype=np.uint32)
    rc = ph._L.ph_gpu_index_stream_u64(idx._h, C.c_void_p(d_keys.data_ptr()), keys.size,
                                       C.c_void_p(h_out.ctypes.data), 4, 1)
    assert rc == ph.E_INVALID
    d_out = torch.zeros(keys.size, dtype=torch.int32, device="cuda")
    rc = ph._L.ph_gpu_index_stream_u64(idx._h, C.c_void_p(d_keys.data_ptr()), keys.size,
                                       C.c_void_p(d_out.data_ptr()), 4, 1)
    assert rc == ph.OK  # both on the device: served without staging
    seq = torch.zeros(8, dtype=torch.int64, device="cuda")
    rc = ph._L.ph_gpu_index_stream_kmers(idx._h, C.c_void_p(seq.data_ptr()), 256, 31,
                                         C.c_void_p(h_out.ctypes.data), 4, 1)
    assert rc == ph.E_INVALID


def test_wrapper_checks_with_device_tensors(ph, ref):
    from oracle.bindings import corpus_u64_np
    keys = corpus_u64_np(0, 50_000, 4)
    idx = ph.PtrHashIndex(ref.build_u64(keys, ref.params("default", lambda_=(30, 10))))
    d_keys = torch.from_numpy(keys.view(np.int64)).cuda()
    with pytest.raises(ValueError, match="CUDA tensor"):
        idx.query(d_keys, out=np.zeros(keys.size, dtype=np.uint32))
    with pytest.raises(ValueError, match="byte elements"):
        idx.query(d_keys, out=torch.zeros(keys.size, dtype=torch.int32, device="cuda"),
                  out_width=8)
    with pytest.raises(ValueError, match="64-bit words"):
        idx.query(d_keys.to(torch.int32))
    s = torch.cuda.Stream()
    out = idx.query(d_keys, stream=s)  # torch.cuda.Stream objects are accepted
    s.synchronize()
    assert out.numel() == keys.size


def test_misaligned_device_pointers_are_rejected(ph, ref):
    """A u64 key array not 8-byte aligned (or an output not aligned to its width) is an
    argument error, not a device fault that would poison the context."""
    from oracle.bindings import corpus_u64_np
    keys = corpus_u64_np(0, 20_000, 4)
    idx = ph.PtrHashIndex(ref.build_u64(keys, ref.params("default", lambda_=(30, 10))))
    buf = torch.zeros(keys.size * 8 + 16, dtype=torch.uint8, device="cuda")
    out = torch.zeros(keys.size + 4, dtype=torch.int32, device="cuda")
    rc = ph._L.ph_gpu_query_u64(idx._h, C.c_void_p(buf.data_ptr() + 3), keys.size,
                                C.c_void_p(out.data_ptr()), 4, 1, None)
    assert rc == ph.E_INVALID
    rc = ph._L.ph_gpu_query_u64(idx._h, C.c_void_p(buf.data_ptr()), keys.size,
                                C.c_void_p(out.data_ptr() + 2), 4, 1, None)
    assert rc == ph.E_INVALID
    rc = ph._L.ph_gpu_query_u64(idx._h, C.c_void_p(buf.data_ptr() + 8), keys.size,
                                C.c_void_p(out.data_ptr() + 4), 4, 1, None)
    assert rc == ph.OK  # 8-B / 4-B aligned (not 16-B): served
    torch.cuda.synchronize()
