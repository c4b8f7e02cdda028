"""Python mirror of the reference query API over the C ABI (include/ph_gpu.h).

``PtrHashIndex`` keeps the reference's method names and meaning
(/root/reference/proj/include/ptrhash/index.hpp:58-81):

  index(key) / index_no_remap(key)                    single key   (index.hpp:60-64)
  index_loop / index_batched / index_stream(keys, ...) bulk queries (index.hpp:72-81)

``keys`` may be a CUDA ``torch.Tensor`` (device-resident, asynchronous on the
current torch stream), a CPU tensor / numpy array (host-resident: pipelined
H2D -> kernel -> D2H inside the library, synchronous), or — for string
indexes — a ``(bytes_buffer, offsets)`` pair in either residence. The
``lookahead`` / ``batch_size`` arguments are accepted for signature parity and
ignored: the GPU kernel has its own latency hiding.

There is no CPU fallback: if libph_gpu.so is missing this module raises on import.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# PH_GPU_LIB: a tuning build of the same library (tools/; paper_2502_15539_b200/variants/)
LIB_PATH = os.environ.get("PH_GPU_LIB") or os.path.join(_HERE, "libph_gpu.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -m paper_2502_15539_b200.build` "
        "(the query path has no CPU fallback)")

_L = C.CDLL(LIB_PATH)
u8p = C.POINTER(C.c_uint8)
u64p = C.POINTER(C.c_uint64)


class Info(C.Structure):
    _fields_ = [
        ("n", C.c_uint64), ("parts", C.c_uint64), ("slots_per_part", C.c_uint64),
        ("buckets_per_part", C.c_uint64), ("seed", C.c_uint64), ("pilot_bytes", C.c_uint64),
        ("remap_values", C.c_uint64), ("remap_bytes", C.c_uint64),
        ("key_kind", C.c_uint8), ("hash_algo", C.c_uint8), ("bucket_fn", C.c_uint8),
        ("remap_kind", C.c_uint8), ("reduce_kind", C.c_uint8), ("pow2", C.c_uint8),
        ("device", C.c_int32),
    ]


_L.ph_gpu_last_error.restype = C.c_char_p
_L.ph_gpu_index_create.argtypes = [u8p, C.c_size_t, C.c_int, C.POINTER(C.c_void_p)]
_L.ph_gpu_index_destroy.argtypes = [C.c_void_p]
_L.ph_gpu_index_info.argtypes = [C.c_void_p, C.POINTER(Info)]
_L.ph_gpu_query_u64.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_int, C.c_int,
                                C.c_void_p]
_L.ph_gpu_query_bytes.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p,
                                  C.c_int, C.c_int, C.c_void_p]
_L.ph_gpu_index_stream_u64.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_int,
                                       C.c_int]
_L.ph_gpu_index_stream_bytes.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t,
                                         C.c_void_p, C.c_int, C.c_int]
_L.ph_gpu_query_kmers.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_int, C.c_void_p,
                                  C.c_int, C.c_int, C.c_void_p]
_L.ph_gpu_index_stream_kmers.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_int, C.c_void_p,
                                         C.c_int, C.c_int]
_L.ph_gpu_index_u64.argtypes = [C.c_void_p, C.c_uint64, C.c_int, u64p]
_L.ph_gpu_index_bytes.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, u64p]
_L.ph_gpu_launch_count.restype = C.c_uint64
_L.ph_gpu_index_load.argtypes = [C.c_char_p, C.c_int, C.POINTER(C.c_void_p)]
_L.ph_gpu_verify_bijection.argtypes = [C.c_void_p, C.c_size_t, C.c_int, C.c_uint64, C.c_int,
                                       u64p, u64p]
_L.ph_gpu_set_launch.argtypes = [C.c_int, C.c_int]
_L.ph_gpu_set_partition.argtypes = [C.c_int]
_L.ph_gpu_set_regime.argtypes = [C.c_int]
_L.ph_gpu_index_set_l2_policy.argtypes = [C.c_void_p, C.c_uint64, C.c_int]

# status codes (ph_gpu.h)
OK, E_INVALID, E_FORMAT, E_CUDA, E_KEYKIND, E_NOMEM, E_UNSUPPORTED = range(7)


class PhGpuError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class SerdeError(PhGpuError):
    """Malformed PTRH bytes (the reference's SerdeError, serde.hpp:39-42)."""


def _check(rc: int):
    if rc != OK:
        msg = _L.ph_gpu_last_error().decode()
        if rc == E_FORMAT:
            raise SerdeError(rc, msg)
        raise PhGpuError(rc, msg)


def launch_count() -> int:
    """Query-kernel launches made by this process through libph_gpu.so."""
    return int(_L.ph_gpu_launch_count())


def set_launch(threads_per_block: int = 0, blocks_per_sm: int = 0):
    _check(_L.ph_gpu_set_launch(threads_per_block, blocks_per_sm))


def set_partition(mode: int):
    """0 automatic, 1 never, 2 whenever the index allows (ph_gpu_set_partition)."""
    _check(_L.ph_gpu_set_partition(mode))


def set_regime(regime: int):
    _check(_L.ph_gpu_set_regime(regime))


_L.ph_gpu_set_pass_timing.argtypes = [C.c_int]
_L.ph_gpu_pass_times.argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_int)]


_L.ph_gpu_index_trim.argtypes = [C.c_void_p]
_L.ph_gpu_bucket_sizes.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_size_t,
                                   C.POINTER(C.c_size_t)]
_L.ph_gpu_build_prepare_u64.argtypes = [C.c_void_p, C.c_size_t, C.c_uint64, C.c_uint64,
                                        C.c_uint64, C.c_int, C.c_void_p, C.c_void_p,
                                        C.POINTER(C.c_int)]


def build_prepare_u64(keys, parts: int, slots_per_part: int, seed: int, device: int = 0):
    """Construction assist (ph_gpu_build_prepare_u64): the hashes of the CUDA u64 tensor
    `keys` in part-major, per-part-sorted order, the part offsets, and the status
    (0 ok, 1 oversubscribed part, 2 duplicate hashes)."""
    import torch
    n = keys.numel()
    hashes = torch.empty(n, dtype=torch.int64, device=keys.device)
    offsets = torch.empty(parts + 1, dtype=torch.int64, device=keys.device)
    st = C.c_int(0)
    _check(_L.ph_gpu_build_prepare_u64(C.c_void_p(keys.data_ptr() if n else 0), n, parts,
                                       slots_per_part, seed, device,
                                       C.c_void_p(hashes.data_ptr() if n else 0),
                                       C.c_void_p(offsets.data_ptr()), C.byref(st)))
    return hashes, offsets, st.value


def set_pass_timing(on: bool):
    """Record CUDA events around the partitioned path's passes (profiling aid)."""
    _check(_L.ph_gpu_set_pass_timing(1 if on else 0))


def pass_times():
    """(summed ms of bin, query, unbin passes, number of timed calls) since set_pass_timing."""
    ms = (C.c_double * 3)()
    calls = C.c_int(0)
    _check(_L.ph_gpu_pass_times(ms, C.byref(calls)))
    return [ms[0], ms[1], ms[2]], calls.value


def _is_torch(x):
    return type(x).__module__.startswith("torch")


def _stream_ptr(stream):
    if stream is not None:
        return C.c_void_p(int(stream))
    import torch
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


class PtrHashIndex:
    """GPU-resident PtrHash index built from the reference's PTRH v1 bytes."""

    def __init__(self, ptrh: bytes, device: int = 0):
        buf = (C.c_uint8 * len(ptrh)).from_buffer_copy(ptrh) if len(ptrh) else (C.c_uint8 * 1)()
        h = C.c_void_p()
        _check(_L.ph_gpu_index_create(C.cast(buf, u8p), len(ptrh), device, C.byref(h)))
        self._h = h
        info = Info()
        _check(_L.ph_gpu_index_info(h, C.byref(info)))
        self.info = info

    @classmethod
    def load(cls, path: str, device: int = 0) -> "PtrHashIndex":
        """load_index (serde.cpp:251-260): mmap + pinned upload (ph_gpu_index_load)."""
        self = cls.__new__(cls)
        h = C.c_void_p()
        _check(_L.ph_gpu_index_load(os.fsencode(path), device, C.byref(h)))
        self._h = h
        info = Info()
        _check(_L.ph_gpu_index_info(h, C.byref(info)))
        self.info = info
        return self

    def verify_bijection(self, out, n=None) -> tuple:
        """(out_of_range, duplicates) of device outputs, verify_bijection (ptrhash.cpp:186-210)."""
        oob, dup = C.c_uint64(), C.c_uint64()
        _check(_L.ph_gpu_verify_bijection(C.c_void_p(out.data_ptr()), out.numel(),
                                          out.element_size(), int(self.info.n if n is None else n),
                                          int(self.info.device), C.byref(oob), C.byref(dup)))
        return int(oob.value), int(dup.value)

    def bucket_sizes(self, keys):
        """ph_gpu_bucket_sizes: hist[s] = number of buckets holding s of the keys (CUDA u64
        tensor); for the build's key set this is the reference's bucket_size_counts."""
        import numpy as np
        cap = 4096
        hist = np.zeros(cap, dtype=np.uint64)
        ln = C.c_size_t(0)
        _check(_L.ph_gpu_bucket_sizes(self._h, C.c_void_p(keys.data_ptr()), keys.numel(),
                                      C.c_void_p(hist.ctypes.data), cap, C.byref(ln)))
        return hist[: min(ln.value, cap)].copy()

    def trim(self):
        """Release the index's cached per-call scratch (ph_gpu_index_trim)."""
        _check(_L.ph_gpu_index_trim(self._h))

    def set_l2_policy(self, hot_bytes: int, flags: int = 0):
        """Pilot layout / L2 policy (ph_gpu_index_set_l2_policy); results are unaffected."""
        _check(_L.ph_gpu_index_set_l2_policy(self._h, hot_bytes, flags))

    def close(self):
        if getattr(self, "_h", None):
            _L.ph_gpu_index_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- properties mirroring PtrHashIndex accessors (index.hpp:48-58) ----
    def n(self) -> int:
        return int(self.info.n)

    def seed(self) -> int:
        return int(self.info.seed)

    def shape(self):
        return (int(self.info.n), int(self.info.parts), int(self.info.slots_per_part),
                int(self.info.buckets_per_part))

    @property
    def key_kind(self) -> int:
        return int(self.info.key_kind)

    # ---- single key (index.hpp:60-64) ----
    def index(self, key) -> int:
        return self._single(key, True)

    def index_no_remap(self, key) -> int:
        return self._single(key, False)

    def _single(self, key, minimal: bool) -> int:
        out = C.c_uint64()
        if isinstance(key, (bytes, bytearray, str)):
            b = key.encode() if isinstance(key, str) else bytes(key)
            arr = (C.c_uint8 * max(1, len(b))).from_buffer_copy(b if b else b"\0")
            _check(_L.ph_gpu_index_bytes(self._h, arr, len(b), int(minimal), C.byref(out)))
        else:
            _check(_L.ph_gpu_index_u64(self._h, int(key) & (2**64 - 1), int(minimal),
                                       C.byref(out)))
        return int(out.value)

    # ---- bulk (index.hpp:72-81) ----
    def index_loop(self, keys, out=None, minimal=True, out_width=8, stream=None):
        return self.query(keys, out, minimal, out_width, stream)

    def index_batched(self, keys, batch_size=64, out=None, minimal=True, out_width=8,
                      stream=None):
        return self.query(keys, out, minimal, out_width, stream)

    def index_stream(self, keys, lookahead=32, out=None, minimal=True, out_width=8,
                     stream=None):
        return self.query(keys, out, minimal, out_width, stream)

    def query(self, keys, out=None, minimal=True, out_width=4, stream=None):
        """out[i] = index(keys[i]) (minimal) or index_no_remap(keys[i])."""
        if out_width not in (4, 8):
            raise ValueError("out_width must be 4 or 8")
        if isinstance(keys, tuple):
            return self._query_bytes(keys[0], keys[1], out, minimal, out_width, stream)
        if _is_torch(keys) and keys.is_cuda:
            import torch
            n = keys.numel()
            if out is None:
                out = torch.empty(n, dtype=torch.int32 if out_width == 4 else torch.int64,
                                  device=keys.device)
            assert keys.is_contiguous() and out.is_contiguous() and out.numel() >= n
            _check(_L.ph_gpu_query_u64(self._h, C.c_void_p(keys.data_ptr()), n,
                                       C.c_void_p(out.data_ptr()), out_width, int(minimal),
                                       _stream_ptr(stream)))
            return out
        k = keys.numpy() if _is_torch(keys) else keys
        k = np.ascontiguousarray(k).view(np.uint64) if k.dtype != np.uint64 else np.ascontiguousarray(k)
        if out is None:
            out = np.empty(k.size, dtype=np.uint32 if out_width == 4 else np.uint64)
        o = out.numpy() if _is_torch(out) else out
        _check(_L.ph_gpu_index_stream_u64(self._h, C.c_void_p(k.ctypes.data), k.size,
                                          C.c_void_p(o.ctypes.data), out_width, int(minimal)))
        return out

    def query_kmers(self, seq, n_bases: int, k: int = 31, out=None, minimal=True, out_width=4,
                    stream=None):
        """Fused k-mer queries: out[i] = index(kmer_i(seq)) for i < n_bases-k+1 (ph_gpu.h
        ph_gpu_query_kmers). `seq` is the 2-bit packed MSB-first sequence (u64 words)."""
        n = max(0, n_bases - k + 1)
        if _is_torch(seq) and seq.is_cuda:
            import torch
            if out is None:
                out = torch.empty(n, dtype=torch.int32 if out_width == 4 else torch.int64,
                                  device=seq.device)
            _check(_L.ph_gpu_query_kmers(self._h, C.c_void_p(seq.data_ptr()), n_bases, k,
                                         C.c_void_p(out.data_ptr()), out_width, int(minimal),
                                         _stream_ptr(stream)))
            return out
        s = seq.numpy() if _is_torch(seq) else np.ascontiguousarray(seq)
        if out is None:
            out = np.empty(n, dtype=np.uint32 if out_width == 4 else np.uint64)
        o = out.numpy() if _is_torch(out) else out
        _check(_L.ph_gpu_index_stream_kmers(self._h, C.c_void_p(s.ctypes.data), n_bases, k,
                                            C.c_void_p(o.ctypes.data), out_width, int(minimal)))
        return out

    def _query_bytes(self, data, offsets, out, minimal, out_width, stream):
        if _is_torch(data) and data.is_cuda:
            import torch
            n = offsets.numel() - 1
            if out is None:
                out = torch.empty(n, dtype=torch.int32 if out_width == 4 else torch.int64,
                                  device=data.device)
            _check(_L.ph_gpu_query_bytes(self._h, C.c_void_p(data.data_ptr()),
                                         C.c_void_p(offsets.data_ptr()), n,
                                         C.c_void_p(out.data_ptr()), out_width, int(minimal),
                                         _stream_ptr(stream)))
            return out
        d = data.numpy() if _is_torch(data) else np.ascontiguousarray(data, dtype=np.uint8)
        o_ = offsets.numpy() if _is_torch(offsets) else np.ascontiguousarray(offsets, dtype=np.uint64)
        n = o_.size - 1
        if out is None:
            out = np.empty(n, dtype=np.uint32 if out_width == 4 else np.uint64)
        oo = out.numpy() if _is_torch(out) else out
        if d.size == 0:
            d = np.zeros(1, dtype=np.uint8)
        _check(_L.ph_gpu_index_stream_bytes(self._h, C.c_void_p(d.ctypes.data),
                                            C.c_void_p(o_.ctypes.data), n,
                                            C.c_void_p(oo.ctypes.data), out_width, int(minimal)))
        return out
