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
_L.ph_gpu_index_bytes.argtypes = [C.c_void_p, C.c_char_p, C.c_size_t, C.c_int, u64p]
_L.ph_gpu_launch_count.restype = C.c_uint64
_L.ph_gpu_index_load.argtypes = [C.c_char_p, C.c_int, C.POINTER(C.c_void_p)]
_L.ph_gpu_verify_bijection.argtypes = [C.c_void_p, C.c_size_t, C.c_int, C.c_uint64, C.c_int,
                                       u64p, u64p]
_L.ph_gpu_set_launch.argtypes = [C.c_int, C.c_int]
_L.ph_gpu_set_partition.argtypes = [C.c_int]
_L.ph_gpu_set_regime.argtypes = [C.c_int]
_L.ph_gpu_index_set_l2_policy.argtypes = [C.c_void_p, C.c_uint64, C.c_int]
try:  # (absent from tuning builds of older sources, tools/variant_ab.py)
    _L.ph_gpu_index_set_scratch_limit.argtypes = [C.c_void_p, C.c_uint64]
    _L.ph_gpu_gather_replay_u64.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]
except AttributeError:
    pass

# status codes (ph_gpu.h)
OK, E_INVALID, E_FORMAT, E_CUDA, E_KEYKIND, E_NOMEM, E_UNSUPPORTED, E_DUPLICATE, E_BUILD_FAILED = range(9)


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


# ---- construction: ph_gpu_build_u64 --------------------------------------

BUCKET_FN = {"linear": 0, "quadratic": 1, "cubic": 2, "skewed": 3, "optimal": 4}
REMAP = {"plain32": 0, "cacheline-ef": 1, "clef": 1, "elias-fano": 2, "ef": 2}
REDUCE = {"pow2-mul": 0, "fastmod-single": 1, "fastmod-multi": 2}


class BuildParams(C.Structure):
    """BuildParams (shape.hpp:46-56); parts/slots_per_part/buckets_per_part force a shape."""
    _fields_ = [
        ("alpha_num", C.c_uint32), ("alpha_den", C.c_uint32),
        ("lambda_num", C.c_uint32), ("lambda_den", C.c_uint32),
        ("bucket_fn", C.c_uint8), ("remap_kind", C.c_uint8), ("reduce_kind", C.c_uint8),
        ("reserved", C.c_uint8), ("max_seed_retries", C.c_uint32), ("seed", C.c_uint64),
        ("parts", C.c_uint64), ("slots_per_part", C.c_uint64), ("buckets_per_part", C.c_uint64),
    ]


class BuildStats(C.Structure):
    """BuildStats (build.hpp:10-45) plus per-stage wall times."""
    _fields_ = [
        ("n", C.c_uint64), ("parts", C.c_uint64), ("slots_per_part", C.c_uint64),
        ("buckets_per_part", C.c_uint64), ("seed", C.c_uint64), ("attempts", C.c_uint32),
        ("remap_kind", C.c_uint8), ("remap_fell_back", C.c_uint8), ("reserved", C.c_uint8 * 2),
        ("total_evictions", C.c_uint64), ("evictions_by_percentile", C.c_uint64 * 100),
        ("pilot_bytes", C.c_uint64), ("remap_payload_bytes", C.c_uint64),
        ("upload_ms", C.c_double), ("prepare_ms", C.c_double), ("search_ms", C.c_double),
        ("remap_ms", C.c_double), ("total_ms", C.c_double),
    ]

    def as_dict(self) -> dict:
        d = {k: getattr(self, k) for k, _ in self._fields_ if k not in ("reserved", "evictions_by_percentile")}
        d["evictions_by_percentile"] = list(self.evictions_by_percentile)
        d["search_on_gpu"] = bool(self.reserved[0])
        return d


_L.ph_build_preset.argtypes = [C.c_char_p, C.POINTER(BuildParams)]
_L.ph_build_compute_shape.argtypes = [C.c_uint64, C.POINTER(BuildParams), u64p, u64p, u64p]
_L.ph_gpu_build_u64.argtypes = [C.c_void_p, C.c_size_t, C.POINTER(BuildParams), C.c_uint, C.c_int,
                                C.POINTER(u8p), C.POINTER(C.c_size_t), C.POINTER(BuildStats)]
_L.ph_build_from_sorted_u64.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.POINTER(BuildParams),
                                        C.c_uint64, C.c_uint, C.POINTER(u8p),
                                        C.POINTER(C.c_size_t), C.POINTER(BuildStats)]
_L.ph_free.argtypes = [C.c_void_p]
_L.ph_gpu_set_build_search.argtypes = [C.c_int]


def set_build_search(mode: int):
    """Where build_u64 runs the pilot search: 0 GPU with host fallback (default), 1 host
    threads, 2 GPU or PhGpuError(E_UNSUPPORTED)."""
    _check(_L.ph_gpu_set_build_search(mode))


def build_params(preset="default", *, lambda_=None, alpha=None, bucket_fn=None, remap=None,
                 reduce=None, seed=None, retries=None, shape=None) -> BuildParams:
    """preset() (shape.cpp:65-84) with the same overrides as the reference's BuildParams."""
    p = BuildParams()
    _check(_L.ph_build_preset(preset.encode(), C.byref(p)))
    if lambda_ is not None:
        p.lambda_num, p.lambda_den = lambda_
    if alpha is not None:
        p.alpha_num, p.alpha_den = alpha
    if bucket_fn is not None:
        p.bucket_fn = BUCKET_FN[bucket_fn] if isinstance(bucket_fn, str) else bucket_fn
    if remap is not None:
        p.remap_kind = REMAP[remap] if isinstance(remap, str) else remap
    if reduce is not None:
        p.reduce_kind = REDUCE[reduce] if isinstance(reduce, str) else reduce
    if seed is not None:
        p.seed = seed
    if retries is not None:
        p.max_seed_retries = retries
    if shape is not None:
        p.parts, p.slots_per_part, p.buckets_per_part = shape
    return p


def compute_shape(n: int, params: BuildParams):
    P, S, B = C.c_uint64(), C.c_uint64(), C.c_uint64()
    _check(_L.ph_build_compute_shape(n, C.byref(params), C.byref(P), C.byref(S), C.byref(B)))
    return P.value, S.value, B.value


def _take_ptrh(ptr, ln) -> bytes:
    try:
        return C.string_at(ptr, ln.value)
    finally:
        _L.ph_free(ptr)


def build_u64(keys, params: BuildParams | None = None, threads: int = 0, device: int = 0,
              stats: bool = False):
    """build(keys, params, threads) + serialize() (construction.cpp:139-143): PTRH v1 bytes.
    `keys` is a numpy u64 array (host) or a CUDA int64/uint64 tensor (device)."""
    params = params if params is not None else build_params()
    if _is_torch(keys):
        if _dtype_name(keys) not in ("int64", "uint64") or not _contiguous(keys):
            raise ValueError("keys must be a contiguous int64/uint64 tensor")
        ptr, n = (keys.data_ptr() if keys.numel() else None), keys.numel()
    else:
        keys = np.ascontiguousarray(keys)
        if keys.dtype not in (np.uint64, np.int64):
            raise ValueError("keys must be a uint64/int64 array")
        ptr, n = (keys.ctypes.data if keys.size else None), keys.size
    out, ln, st = u8p(), C.c_size_t(0), BuildStats()
    _check(_L.ph_gpu_build_u64(C.c_void_p(ptr), n, C.byref(params), threads, device, C.byref(out),
                               C.byref(ln), C.byref(st)))
    b = _take_ptrh(out, ln)
    return (b, st.as_dict()) if stats else b


_L.ph_gpu_build_bytes.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.POINTER(BuildParams), C.c_int,
                                  C.c_uint, C.c_int, C.POINTER(u8p), C.POINTER(C.c_size_t),
                                  C.POINTER(BuildStats)]


def build_bytes(data, offsets, params: BuildParams | None = None, hash_algo: int = 1, threads: int = 0,
                device: int = 0, stats: bool = False):
    """build(span<const std::string>) + serialize() (construction.cpp:154-226) for keys given as
    concatenated bytes `data` (numpy u8 or CUDA uint8 tensor) + u64 `offsets[n+1]`: PTRH v1
    bytes of a string-key index hashed with aes64 (1) or portable64 (3)."""
    params = params if params is not None else build_params()
    if _is_torch(data):
        n = offsets.numel() - 1
        dp, op = data.data_ptr(), offsets.data_ptr()
    else:
        data = np.ascontiguousarray(data, dtype=np.uint8)
        offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        n = offsets.size - 1
        dp, op = (data.ctypes.data if data.size else None), offsets.ctypes.data
    out, ln, st = u8p(), C.c_size_t(0), BuildStats()
    _check(_L.ph_gpu_build_bytes(C.c_void_p(dp), C.c_void_p(op), n, C.byref(params), hash_algo, threads,
                                 device, C.byref(out), C.byref(ln), C.byref(st)))
    b = _take_ptrh(out, ln)
    return (b, st.as_dict()) if stats else b


def build_from_sorted_u64(hashes: np.ndarray, offsets: np.ndarray, params: BuildParams, seed: int,
                          threads: int = 0, stats: bool = False):
    """The host stage of one build attempt (no GPU): sorted part-major hashes + part offsets
    -> PTRH bytes, or PhGpuError(E_BUILD_FAILED) if a part cannot be placed."""
    hashes = np.ascontiguousarray(hashes, dtype=np.uint64)
    offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
    out, ln, st = u8p(), C.c_size_t(0), BuildStats()
    _check(_L.ph_build_from_sorted_u64(C.c_void_p(hashes.ctypes.data), C.c_void_p(offsets.ctypes.data),
                                       hashes.size, C.byref(params), seed, threads, C.byref(out),
                                       C.byref(ln), C.byref(st)))
    b = _take_ptrh(out, ln)
    return (b, st.as_dict()) if stats else b


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
    """None (torch's current stream), a torch.cuda.Stream, or a raw cudaStream_t (int)."""
    if stream is None:
        import torch
        return C.c_void_p(torch.cuda.current_stream().cuda_stream)
    if hasattr(stream, "cuda_stream"):
        return C.c_void_p(stream.cuda_stream)
    return C.c_void_p(int(stream))


_WORD_DTYPES = ("int64", "uint64")


def _dtype_name(x) -> str:
    return str(x.dtype).replace("torch.", "")


def _contiguous(x) -> bool:
    return x.is_contiguous() if _is_torch(x) else bool(x.flags["C_CONTIGUOUS"])


def _count(x) -> int:
    return x.numel() if _is_torch(x) else x.size


def _check_words(x, what: str, min_count: int):
    """x: a contiguous 64-bit-word array (torch or numpy) with at least min_count entries."""
    if _dtype_name(x) not in _WORD_DTYPES:
        raise ValueError(f"{what} must hold 64-bit words (int64/uint64), got {x.dtype}")
    if not _contiguous(x):
        raise ValueError(f"{what} must be contiguous")
    if _count(x) < min_count:
        raise ValueError(f"{what} holds {_count(x)} entries, needs {min_count}")


def _check_out(out, n: int, out_width: int, cuda: bool):
    """A caller-supplied output: out_width bytes per element, >= n elements, contiguous and
    in the same residence (device or host) as the inputs."""
    if out_width not in (4, 8):
        raise ValueError("out_width must be 4 or 8")
    if out is None:
        return
    if _is_torch(out):
        if bool(out.is_cuda) != cuda:
            raise ValueError("out must live where the keys live (device or host)")
        size = out.element_size()
    else:
        if cuda:
            raise ValueError("out must be a CUDA tensor for device-resident keys")
        if not isinstance(out, np.ndarray):
            raise ValueError("a host out must be a numpy array or a CPU tensor")
        size = out.itemsize
    if size != out_width:
        raise ValueError(f"out has {size}-byte elements but out_width is {out_width}")
    if _count(out) < n:
        raise ValueError(f"out holds {_count(out)} elements, needs {n}")
    if not _contiguous(out):
        raise ValueError("out must be contiguous")


def _new_out(n: int, out_width: int, like):
    if _is_torch(like) and like.is_cuda:
        import torch
        return torch.empty(n, dtype=torch.int32 if out_width == 4 else torch.int64,
                           device=like.device)
    return np.empty(n, dtype=np.uint32 if out_width == 4 else np.uint64)


def _host(x):
    return x.numpy() if _is_torch(x) else x


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

    def set_scratch_limit(self, nbytes: int):
        """Ceiling on cached per-call scratch (ph_gpu_index_set_scratch_limit)."""
        _check(_L.ph_gpu_index_set_scratch_limit(self._h, int(nbytes)))

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
            _check(_L.ph_gpu_index_bytes(self._h, b, len(b), int(minimal), C.byref(out)))
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
        """out[i] = index(keys[i]) (minimal) or index_no_remap(keys[i]). Raises ValueError
        on a key dtype other than int64/uint64, a non-contiguous array, or an `out` of the
        wrong element width, size or residence."""
        if isinstance(keys, tuple):
            return self._query_bytes(keys[0], keys[1], out, minimal, out_width, stream)
        cuda = _is_torch(keys) and keys.is_cuda
        if not _is_torch(keys):
            keys = np.asarray(keys)
        n = _count(keys)
        _check_words(keys, "keys", n)
        _check_out(out, n, out_width, cuda)
        if out is None:
            out = _new_out(n, out_width, keys)
        if cuda:
            _check(_L.ph_gpu_query_u64(self._h, C.c_void_p(keys.data_ptr()), n,
                                       C.c_void_p(out.data_ptr()), out_width, int(minimal),
                                       _stream_ptr(stream)))
            return out
        k, o = _host(keys), _host(out)
        _check(_L.ph_gpu_index_stream_u64(self._h, C.c_void_p(k.ctypes.data), n,
                                          C.c_void_p(o.ctypes.data), out_width, int(minimal)))
        return out

    def gather_replay(self, keys, stream=None):
        """Measurement: the pilot reads alone at the true bucket addresses of the CUDA u64
        tensor `keys` (ph_gpu_gather_replay_u64; bench.py's replay bound)."""
        if not (_is_torch(keys) and keys.is_cuda):
            raise ValueError("gather_replay takes a CUDA tensor")
        _check_words(keys, "keys", keys.numel())
        _check(_L.ph_gpu_gather_replay_u64(self._h, C.c_void_p(keys.data_ptr()), keys.numel(),
                                           _stream_ptr(stream)))

    def query_kmers(self, seq, n_bases: int, k: int = 31, out=None, minimal=True, out_width=4,
                    stream=None):
        """Fused k-mer queries: out[i] = index(kmer_i(seq)) for i < n_bases-k+1 (ph_gpu.h
        ph_gpu_query_kmers). `seq` is the 2-bit packed MSB-first sequence (u64 words, at
        least ceil(n_bases/32) of them)."""
        if not 1 <= k <= 32:
            raise ValueError("k must be in [1, 32]")
        n = max(0, n_bases - k + 1)
        cuda = _is_torch(seq) and seq.is_cuda
        if not _is_torch(seq):
            seq = np.asarray(seq)
        _check_words(seq, "seq", (n_bases + 31) // 32)
        _check_out(out, n, out_width, cuda)
        if out is None:
            out = _new_out(n, out_width, seq)
        if cuda:
            _check(_L.ph_gpu_query_kmers(self._h, C.c_void_p(seq.data_ptr()), n_bases, k,
                                         C.c_void_p(out.data_ptr()), out_width, int(minimal),
                                         _stream_ptr(stream)))
            return out
        s_, o = _host(seq), _host(out)
        _check(_L.ph_gpu_index_stream_kmers(self._h, C.c_void_p(s_.ctypes.data), n_bases, k,
                                            C.c_void_p(o.ctypes.data), out_width, int(minimal)))
        return out

    def _query_bytes(self, data, offsets, out, minimal, out_width, stream):
        cuda = _is_torch(data) and data.is_cuda
        if (_is_torch(offsets) and offsets.is_cuda) != cuda:
            raise ValueError("bytes and offsets must both be on the device or both on the host")
        if not _is_torch(data):
            data = np.asarray(data)
        if not _is_torch(offsets):
            offsets = np.asarray(offsets)
        if _dtype_name(data) not in ("uint8", "int8"):
            raise ValueError(f"string bytes must be uint8, got {data.dtype}")
        if not _contiguous(data):
            raise ValueError("string bytes must be contiguous")
        if _count(offsets) < 1:
            raise ValueError("offsets must hold n+1 entries")
        n = _count(offsets) - 1
        _check_words(offsets, "offsets", n + 1)
        _check_out(out, n, out_width, cuda)
        if out is None:
            out = _new_out(n, out_width, data)
        if cuda:
            _check(_L.ph_gpu_query_bytes(self._h, C.c_void_p(data.data_ptr()),
                                         C.c_void_p(offsets.data_ptr()), n,
                                         C.c_void_p(out.data_ptr()), out_width, int(minimal),
                                         _stream_ptr(stream)))
            return out
        d, o_, oo = _host(data), _host(offsets), _host(out)
        if d.size == 0:
            d = np.zeros(1, dtype=np.uint8)
        _check(_L.ph_gpu_index_stream_bytes(self._h, C.c_void_p(d.ctypes.data),
                                            C.c_void_p(o_.ctypes.data), n,
                                            C.c_void_p(oo.ctypes.data), out_width, int(minimal)))
        return out
