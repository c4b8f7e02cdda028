"""Argument checks of the Python mirror (paper_2502_15539_b200/ph_gpu.py) that run before any
device call: key / sequence / offsets dtypes and sizes, `out` width, size and residence, and
stream objects. CPU-only (the checks never reach the C ABI when they fail)."""
import numpy as np
import pytest

from paper_2502_15539_b200 import ph_gpu


class _FakeIndex(ph_gpu.PtrHashIndex):
    """A PtrHashIndex whose handle is never used: every call below must fail validation."""

    def __init__(self):
        self._h = None

    def close(self):
        pass


@pytest.fixture()
def idx():
    return _FakeIndex()


def test_key_dtype_rejected(idx):
    with pytest.raises(ValueError, match="64-bit words"):
        idx.query(np.zeros(8, dtype=np.int32))
    with pytest.raises(ValueError, match="64-bit words"):
        idx.query(np.zeros(8, dtype=np.float64))


def test_noncontiguous_keys_rejected(idx):
    with pytest.raises(ValueError, match="contiguous"):
        idx.query(np.zeros(16, dtype=np.uint64)[::2])


@pytest.mark.parametrize("width,dtype", [(8, np.uint32), (4, np.uint64), (4, np.int16)])
def test_out_width_mismatch_rejected(idx, width, dtype):
    with pytest.raises(ValueError, match="byte elements"):
        idx.query(np.zeros(8, dtype=np.uint64), out=np.zeros(8, dtype=dtype), out_width=width)


def test_out_too_small_rejected(idx):
    with pytest.raises(ValueError, match="needs 8"):
        idx.query(np.zeros(8, dtype=np.uint64), out=np.zeros(7, dtype=np.uint32), out_width=4)


def test_out_width_value_rejected(idx):
    with pytest.raises(ValueError, match="out_width"):
        idx.query(np.zeros(8, dtype=np.uint64), out_width=2)


def test_kmer_sequence_checks(idx):
    with pytest.raises(ValueError, match="needs 4"):
        idx.query_kmers(np.zeros(3, dtype=np.uint64), 100, 31)  # ceil(100/32) = 4 words
    with pytest.raises(ValueError, match="64-bit words"):
        idx.query_kmers(np.zeros(4, dtype=np.uint32), 100, 31)
    with pytest.raises(ValueError, match="k must be"):
        idx.query_kmers(np.zeros(4, dtype=np.uint64), 100, 33)


def test_string_argument_checks(idx):
    data = np.frombuffer(b"abcdef", dtype=np.uint8)
    with pytest.raises(ValueError, match="64-bit words"):
        idx.query((data, np.array([0, 3, 6], dtype=np.int32)))
    with pytest.raises(ValueError, match="uint8"):
        idx.query((np.zeros(6, dtype=np.int64), np.array([0, 3, 6], dtype=np.uint64)))
    with pytest.raises(ValueError, match="n\\+1"):
        idx.query((data, np.zeros(0, dtype=np.uint64)))
    with pytest.raises(ValueError, match="needs 2"):
        idx.query((data, np.array([0, 3, 6], dtype=np.uint64)),
                  out=np.zeros(1, dtype=np.uint32), out_width=4)


def test_stream_objects():
    class S:  # a torch.cuda.Stream-like object
        cuda_stream = 1234
    assert ph_gpu._stream_ptr(S()).value == 1234
    assert ph_gpu._stream_ptr(5678).value == 5678
