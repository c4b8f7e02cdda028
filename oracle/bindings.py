"""TEST INFRASTRUCTURE ONLY — ctypes bindings to the two CPU checkers.

* ``Ref``  -> oracle/_ref/libptrhash_ref.so: the unmodified reference C++ library
  (built from /root/reference/proj/src by oracle/Makefile) behind oracle/ref_shim.cpp.
  Used to BUILD indexes (the reference builder, as north_star requires), as the
  bit-exact parity oracle, and as bench.py's reference arm / cpu_baseline.
* ``Port`` -> oracle/_ref/libph_oracle.so: our plain-C restatement (ph_oracle.c),
  pinned against ``Ref`` and tests/golden/.

Only tests/, __graft_entry__.smoke() and bench.py (fixture + CPU baseline legs)
import this module. The product library never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libptrhash_ref.so")
PORT_SO = os.path.join(HERE, "_ref", "libph_oracle.so")

u8p = C.POINTER(C.c_uint8)
u64p = C.POINTER(C.c_uint64)

# ids mirror the PTRH header ids (shape.hpp:23-35, hash.hpp:37-43, reduce.hpp:11-20)
BUCKET_FN = {"linear": 0, "quadratic": 1, "cubic": 2, "skewed": 3, "optimal": 4}
REMAP = {"plain32": 0, "cacheline-ef": 1, "elias-fano": 2}
REDUCE = {"pow2-mul": 0, "fastmod-single": 1, "fastmod-multi": 2}
HASH = {"fx64": 0, "aes64": 1, "aes128": 2, "portable64": 3, "portable128": 4}


class RefParams(C.Structure):
    _fields_ = [
        ("alpha_num", C.c_uint32), ("alpha_den", C.c_uint32),
        ("lambda_num", C.c_uint32), ("lambda_den", C.c_uint32),
        ("bucket_fn", C.c_int32), ("remap_kind", C.c_int32), ("reduce_kind", C.c_int32),
        ("max_seed_retries", C.c_uint32), ("seed", C.c_uint64),
    ]


def _ptr(a, t=u64p):
    return a.ctypes.data_as(t)


class Ref:
    """The reference library (bit-exactness is against this code)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle` (needs /root/reference)")
        L = self.L = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_build_u64.argtypes = [u64p, C.c_size_t, C.POINTER(RefParams), C.c_uint,
                                    C.POINTER(u8p), C.POINTER(C.c_size_t)]
        L.ref_build_u64_shape.argtypes = [u64p, C.c_size_t, C.POINTER(RefParams), C.c_uint64,
                                          C.c_uint64, C.c_uint64, C.c_uint,
                                          C.POINTER(u8p), C.POINTER(C.c_size_t)]
        for f in (L.ref_build_bytes, L.ref_build_bytes_lean):
            f.argtypes = [u8p, u64p, C.c_size_t, C.POINTER(RefParams), C.c_uint,
                          C.POINTER(u8p), C.POINTER(C.c_size_t)]
        L.ref_free.argtypes = [C.c_void_p]
        L.ref_load.argtypes = [u8p, C.c_size_t]
        L.ref_load.restype = C.c_void_p
        L.ref_unload.argtypes = [C.c_void_p]
        L.ref_index_u64.argtypes = [C.c_void_p, C.c_uint64, C.c_int]
        L.ref_index_u64.restype = C.c_uint64
        L.ref_index_bytes1.argtypes = [C.c_void_p, u8p, C.c_size_t, C.c_int]
        L.ref_index_bytes1.restype = C.c_uint64
        L.ref_query_u64.argtypes = [C.c_void_p, u64p, C.c_size_t, u64p, C.c_int, C.c_int,
                                    C.c_size_t, C.c_uint]
        L.ref_query_bytes.argtypes = [C.c_void_p, u8p, u64p, C.c_size_t, u64p, C.c_int,
                                      C.c_int, C.c_size_t, C.c_uint]
        L.ref_strings_new.argtypes = [u8p, u64p, C.c_size_t]
        L.ref_strings_new.restype = C.c_void_p
        L.ref_strings_free.argtypes = [C.c_void_p]
        L.ref_query_strings.argtypes = [C.c_void_p, C.c_void_p, u64p, C.c_int, C.c_int,
                                        C.c_size_t, C.c_uint]
        L.ref_preset.argtypes = [C.c_char_p, C.POINTER(RefParams)]
        L.ref_compute_shape.argtypes = [C.c_uint64, C.POINTER(RefParams), u64p, u64p, u64p]
        for name in ("ref_mix_constant_inverse",):
            getattr(L, name).restype = C.c_uint64
        for name in ("ref_hash_int", "ref_hash_pilot", "ref_reduce", "ref_corpus_u64"):
            f = getattr(L, name)
            f.argtypes = [C.c_uint64, C.c_uint64]
            f.restype = C.c_uint64
        L.ref_gamma.argtypes = [C.c_int, C.c_uint64]
        L.ref_gamma.restype = C.c_uint64
        L.ref_hash_bytes.argtypes = [u8p, C.c_size_t, C.c_uint64, C.c_int, u64p, u64p]
        L.ref_fastmod_magic.argtypes = [C.c_uint64, u64p, u64p]
        L.ref_part_and_bucket.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, u64p, u64p]
        L.ref_clef_encode.argtypes = [u64p, C.c_size_t, u8p]
        L.ref_clef_get.argtypes = [u8p, C.c_size_t]
        L.ref_clef_get.restype = C.c_uint64
        L.ref_build_prepare_u64.argtypes = [u64p, C.c_size_t, C.c_uint64, C.c_uint64,
                                            C.c_uint64, C.c_uint, u64p, u64p]
        L.ref_build_u64_stats.argtypes = [u64p, C.c_size_t, C.POINTER(RefParams), C.c_uint,
                                          C.POINTER(u8p), C.POINTER(C.c_size_t), u64p,
                                          C.c_size_t, C.POINTER(C.c_size_t)]
        L.ref_hw_threads.restype = C.c_uint

    # ---- params / shape ----
    def params(self, preset="default", *, lambda_=None, bucket_fn=None, remap=None,
               reduce=None, alpha=None, seed=None, retries=None) -> RefParams:
        p = RefParams()
        if self.L.ref_preset(preset.encode(), C.byref(p)) != 0:
            raise ValueError(self.err())
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
        return p

    def shape(self, n, params):
        P, S, B = C.c_uint64(), C.c_uint64(), C.c_uint64()
        if self.L.ref_compute_shape(n, C.byref(params), C.byref(P), C.byref(S), C.byref(B)):
            raise ValueError(self.err())
        return P.value, S.value, B.value

    def err(self) -> str:
        return self.L.ref_last_error().decode()

    def _take(self, rc, out, ln) -> bytes:
        if rc != 0:
            raise RuntimeError("reference build failed: " + self.err())
        b = C.string_at(out, ln.value)
        self.L.ref_free(out)
        return b

    # ---- builders (return PTRH v1 bytes, serde.cpp:142-174) ----
    def build_u64(self, keys: np.ndarray, params: RefParams, threads: int = 0) -> bytes:
        keys = np.ascontiguousarray(keys, dtype=np.uint64)
        out, ln = u8p(), C.c_size_t()
        rc = self.L.ref_build_u64(_ptr(keys), keys.size, C.byref(params), threads,
                                  C.byref(out), C.byref(ln))
        return self._take(rc, out, ln)

    def build_u64_stats(self, keys: np.ndarray, params: RefParams, threads: int = 0):
        """build() with BuildStats: (PTRH bytes, bucket_size_counts) (stats.cpp:59-61)."""
        k = np.ascontiguousarray(keys, dtype=np.uint64)
        out, ln = u8p(), C.c_size_t()
        sizes = np.zeros(4096, dtype=np.uint64)
        slen = C.c_size_t()
        rc = self.L.ref_build_u64_stats(_ptr(k), k.size, C.byref(params), threads, C.byref(out),
                                        C.byref(ln), _ptr(sizes), sizes.size, C.byref(slen))
        return self._take(rc, out, ln), sizes[: min(slen.value, sizes.size)].copy()

    def build_u64_shape(self, keys, params, P, S, B, threads=0) -> bytes:
        keys = np.ascontiguousarray(keys, dtype=np.uint64)
        out, ln = u8p(), C.c_size_t()
        rc = self.L.ref_build_u64_shape(_ptr(keys), keys.size, C.byref(params), P, S, B,
                                        threads, C.byref(out), C.byref(ln))
        return self._take(rc, out, ln)

    def build_bytes(self, data: np.ndarray, offsets: np.ndarray, params, threads=0,
                    lean=False) -> bytes:
        data = np.ascontiguousarray(data, dtype=np.uint8)
        offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        n = offsets.size - 1
        out, ln = u8p(), C.c_size_t()
        f = self.L.ref_build_bytes_lean if lean else self.L.ref_build_bytes
        rc = f(_ptr(data, u8p), _ptr(offsets), n, C.byref(params), threads,
               C.byref(out), C.byref(ln))
        return self._take(rc, out, ln)

    # ---- loaded index ----
    def load(self, ptrh: bytes) -> "RefIndex":
        return RefIndex(self, ptrh)

    def hw_threads(self) -> int:
        return int(self.L.ref_hw_threads())

    # ---- primitives ----
    def hash_bytes(self, b: bytes, seed: int, algo: int):
        arr = (C.c_uint8 * max(1, len(b))).from_buffer_copy(b if b else b"\0")
        hi, lo = C.c_uint64(), C.c_uint64()
        self.L.ref_hash_bytes(C.cast(arr, u8p), len(b), seed, algo, C.byref(hi), C.byref(lo))
        return hi.value, lo.value

    def part_and_bucket(self, h, P, B, fn):
        a, b = C.c_uint64(), C.c_uint64()
        self.L.ref_part_and_bucket(h, P, B, fn, C.byref(a), C.byref(b))
        return a.value, b.value

    def fastmod_magic(self, S):
        a, b = C.c_uint64(), C.c_uint64()
        self.L.ref_fastmod_magic(S, C.byref(a), C.byref(b))
        return a.value, b.value

    def clef_encode(self, values):
        v = np.ascontiguousarray(values, dtype=np.uint64)
        out = (C.c_uint8 * 64)()
        st = self.L.ref_clef_encode(_ptr(v), v.size, C.cast(out, u8p))
        return st, bytes(out)

    def clef_get(self, block: bytes, i: int) -> int:
        arr = (C.c_uint8 * 64).from_buffer_copy(block)
        return self.L.ref_clef_get(C.cast(arr, u8p), i)

    # ---- construction front phases (hash_all, scatter_to_parts, per-part sort) ----
    def build_prepare_u64(self, keys, P: int, S: int, seed: int, threads: int = 0):
        """The reference's own hash_all + scatter_to_parts + per-part std::sort
        (construction.cpp:98-111, engine.hpp:412-518): (hashes, offsets, status) with status
        0 ok, 1 kOversubscribed, 2 kDuplicateHashes."""
        k = np.ascontiguousarray(keys, dtype=np.uint64)
        h = np.empty(k.size, dtype=np.uint64)
        off = np.empty(P + 1, dtype=np.uint64)
        st = self.L.ref_build_prepare_u64(_ptr(k), k.size, P, S, seed, threads, _ptr(h), _ptr(off))
        if st < 0:
            raise RuntimeError(self.err())
        return h, off, st


class RefIndex:
    """A reference PtrHashIndex deserialized from PTRH bytes (serde.cpp:176-240)."""

    MODES = {"loop": 0, "batched": 1, "stream": 2, "single": 3}

    def __init__(self, ref: Ref, ptrh: bytes):
        self.ref = ref
        self._buf = (C.c_uint8 * len(ptrh)).from_buffer_copy(ptrh)
        self.h = ref.L.ref_load(C.cast(self._buf, u8p), len(ptrh))
        if not self.h:
            raise ValueError("reference deserialize failed: " + ref.err())

    def close(self):
        if self.h:
            self.ref.L.ref_unload(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def index(self, key: int, minimal=True) -> int:
        return self.ref.L.ref_index_u64(self.h, key, int(minimal))

    def query_u64(self, keys, minimal=True, mode="stream", width=32, threads=1, out=None):
        keys = np.ascontiguousarray(keys, dtype=np.uint64)
        if out is None:
            out = np.empty(keys.size, dtype=np.uint64)
        rc = self.ref.L.ref_query_u64(self.h, _ptr(keys), keys.size, _ptr(out), int(minimal),
                                      self.MODES[mode], width, threads)
        if rc:
            raise RuntimeError(self.ref.err())
        return out

    def query_bytes(self, data, offsets, minimal=True, mode="single", width=32, threads=1,
                    out=None):
        data = np.ascontiguousarray(data, dtype=np.uint8)
        offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        n = offsets.size - 1
        if out is None:
            out = np.empty(n, dtype=np.uint64)
        rc = self.ref.L.ref_query_bytes(self.h, _ptr(data, u8p), _ptr(offsets), n, _ptr(out),
                                        int(minimal), self.MODES[mode], width, threads)
        if rc:
            raise RuntimeError(self.ref.err())
        return out


class RefStrings:
    """std::string keys materialised once (ref_strings_new), for timing the reference's
    span<const std::string> bulk queries without the string construction."""

    def __init__(self, ref: Ref, data, offsets):
        data = np.ascontiguousarray(data, dtype=np.uint8)
        offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        self.ref, self.n = ref, offsets.size - 1
        self.h = ref.L.ref_strings_new(_ptr(data, u8p), _ptr(offsets), self.n)
        if not self.h:
            raise MemoryError(ref.err())

    def query(self, ri: "RefIndex", minimal=True, mode="stream", width=32, threads=1, out=None):
        if out is None:
            out = np.empty(self.n, dtype=np.uint64)
        rc = self.ref.L.ref_query_strings(ri.h, self.h, _ptr(out), int(minimal),
                                          RefIndex.MODES[mode], width, threads)
        if rc:
            raise RuntimeError(self.ref.err())
        return out

    def close(self):
        if self.h:
            self.ref.L.ref_strings_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class PhoIndex(C.Structure):
    _fields_ = [
        ("key_kind", C.c_uint8), ("hash_algo", C.c_uint8), ("bucket_fn", C.c_uint8),
        ("remap_kind", C.c_uint8), ("reduce_kind", C.c_uint8),
        ("n", C.c_uint64), ("P", C.c_uint64), ("S", C.c_uint64), ("B", C.c_uint64),
        ("seed", C.c_uint64),
        ("pilots", u8p), ("remap", u8p), ("remap_len", C.c_uint64),
        ("ef_count", C.c_uint64), ("ef_universe", C.c_uint64), ("ef_low_bits", C.c_uint8),
        ("ef_low", u64p), ("ef_high", u64p), ("ef_samples", u64p),
        ("ef_low_n", C.c_uint64), ("ef_high_n", C.c_uint64), ("ef_samples_n", C.c_uint64),
        ("magic_hi", C.c_uint64), ("magic_lo", C.c_uint64), ("pow2", C.c_int),
    ]


class Port:
    """Our plain-C restatement of the query path (oracle/ph_oracle.c)."""

    def __init__(self, path: str = PORT_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle port`")
        L = self.L = C.CDLL(path)
        for name in ("pho_mul_hi", "pho_hash_int", "pho_hash_pilot", "pho_reduce",
                     "pho_corpus_u64"):
            f = getattr(L, name)
            f.argtypes = [C.c_uint64, C.c_uint64]
            f.restype = C.c_uint64
        L.pho_mix64.argtypes = [C.c_uint64]
        L.pho_mix64.restype = C.c_uint64
        L.pho_gamma.argtypes = [C.c_int, C.c_uint64]
        L.pho_gamma.restype = C.c_uint64
        L.pho_optimal_table.restype = u64p
        L.pho_fastmod_magic.argtypes = [C.c_uint64, u64p, u64p]
        L.pho_part_and_bucket.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, u64p, u64p]
        L.pho_clef_get.argtypes = [u8p, C.c_size_t]
        L.pho_clef_get.restype = C.c_uint64
        L.pho_hash_bytes.argtypes = [u8p, C.c_size_t, C.c_uint64, C.c_int, u64p, u64p]
        L.pho_parse.argtypes = [u8p, C.c_size_t, C.POINTER(PhoIndex), C.POINTER(C.c_char_p)]
        L.pho_release.argtypes = [C.POINTER(PhoIndex)]
        L.pho_index_u64.argtypes = [C.POINTER(PhoIndex), C.c_uint64, C.c_int]
        L.pho_index_u64.restype = C.c_uint64
        L.pho_query_u64.argtypes = [C.POINTER(PhoIndex), u64p, C.c_size_t, u64p, C.c_int]
        L.pho_query_bytes.argtypes = [C.POINTER(PhoIndex), u8p, u64p, C.c_size_t, u64p, C.c_int]
        L.pho_feistel_perm.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        L.pho_feistel_perm.restype = C.c_uint64
        L.pho_gen_corpus.argtypes = [u64p, C.c_uint64, C.c_uint64, C.c_uint64]
        L.pho_gen_perm_keys.argtypes = [u64p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64,
                                        C.c_uint64]
        L.pho_gen_sample_keys.argtypes = list(L.pho_gen_perm_keys.argtypes)
        L.pho_gen_dna.argtypes = [u64p, C.c_uint64, C.c_uint64, C.c_uint64]
        L.pho_kmers.argtypes = [u64p, C.c_uint64, C.c_int, C.c_uint64, C.c_uint64, u64p]

    def _threaded(self, count, T, fn):
        import threading
        T = T or (os.cpu_count() or 1)
        step = (count + T - 1) // T
        ths = [threading.Thread(target=fn, args=(t * step, min(step, count - t * step)))
               for t in range(T) if t * step < count]
        for th in ths:
            th.start()
        for th in ths:
            th.join()

    def gen_strings(self, start: int, count: int, n: int, seed: int, perm_seed: int = 0,
                    threads: int = 0):
        """Config-4 strings start..start+count (src = Feistel perm if perm_seed) as one
        concatenated byte buffer + u64 offsets[count+1] (ph_oracle.c pho_gen_strings)."""
        import threading
        self.L.pho_gen_strings.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64,
                                           C.c_uint64, u8p, u64p, C.c_uint64]
        self.L.pho_gen_strings.restype = C.c_uint64
        T = threads or (os.cpu_count() or 1)
        step = (count + T - 1) // T
        parts = [None] * T

        def work(t):
            b = t * step
            m = min(step, count - b)
            if m <= 0:
                parts[t] = (np.zeros(0, np.uint8), np.zeros(1, np.uint64))
                return
            data = np.empty(m * 64, dtype=np.uint8)
            offs = np.empty(m + 1, dtype=np.uint64)
            end = self.L.pho_gen_strings(start + b, m, n, seed, perm_seed,
                                         data.ctypes.data_as(u8p), offs.ctypes.data_as(u64p), 0)
            parts[t] = (data[:end], offs)

        ths = [threading.Thread(target=work, args=(t,)) for t in range(T)]
        for th in ths:
            th.start()
        for th in ths:
            th.join()
        total = sum(p[0].size for p in parts)
        data = np.empty(max(total, 1), dtype=np.uint8)
        offs = np.empty(count + 1, dtype=np.uint64)
        pos, k = 0, 0
        for d, o in parts:
            m = o.size - 1
            data[pos:pos + d.size] = d
            offs[k:k + m + 1] = o + np.uint64(pos)
            pos += d.size
            k += m
        return data, offs

    def gen_dna(self, n_bases: int, seed: int, threads: int = 0) -> np.ndarray:
        """2-bit packed MSB-first random sequence (ph_gpu.h layout), ceil(n/32) words."""
        nw = (n_bases + 31) // 32
        out = np.empty(nw, dtype=np.uint64)
        self._threaded(nw, threads, lambda b, m: self.L.pho_gen_dna(
            out[b:].ctypes.data_as(u64p), b, m, seed))
        return out

    def kmers(self, seq: np.ndarray, n_bases: int, k: int, threads: int = 0) -> np.ndarray:
        n = n_bases - k + 1
        out = np.empty(max(n, 0), dtype=np.uint64)
        seq = np.ascontiguousarray(seq, dtype=np.uint64)
        self._threaded(n, threads, lambda b, m: self.L.pho_kmers(
            seq.ctypes.data_as(u64p), n_bases, k, b, m, out[b:].ctypes.data_as(u64p)))
        return out

    def gen_keys(self, kind: str, start: int, count: int, n: int, gen_seed: int, seed: int = 0,
                 threads: int = 0) -> np.ndarray:
        """Host generation of the synthetic key streams ("corpus", "perm", "sample"), threaded."""
        import threading
        out = np.empty(count, dtype=np.uint64)
        T = threads or (os.cpu_count() or 1)
        step = (count + T - 1) // T

        def work(t):
            b = t * step
            m = min(step, count - b)
            if m <= 0:
                return
            ptr = out[b:].ctypes.data_as(u64p)
            if kind == "corpus":
                self.L.pho_gen_corpus(ptr, start + b, m, gen_seed)
            elif kind == "perm":
                self.L.pho_gen_perm_keys(ptr, start + b, m, n, gen_seed, seed)
            else:
                self.L.pho_gen_sample_keys(ptr, start + b, m, n, gen_seed, seed)

        ths = [threading.Thread(target=work, args=(t,)) for t in range(T)]
        for th in ths:
            th.start()
        for th in ths:
            th.join()
        return out

    def hash_bytes(self, b: bytes, seed: int, algo: int):
        arr = (C.c_uint8 * max(1, len(b))).from_buffer_copy(b if b else b"\0")
        hi, lo = C.c_uint64(), C.c_uint64()
        self.L.pho_hash_bytes(C.cast(arr, u8p), len(b), seed, algo, C.byref(hi), C.byref(lo))
        return hi.value, lo.value

    def part_and_bucket(self, h, P, B, fn):
        a, b = C.c_uint64(), C.c_uint64()
        self.L.pho_part_and_bucket(h, P, B, fn, C.byref(a), C.byref(b))
        return a.value, b.value

    def fastmod_magic(self, S):
        a, b = C.c_uint64(), C.c_uint64()
        self.L.pho_fastmod_magic(S, C.byref(a), C.byref(b))
        return a.value, b.value

    def clef_get(self, block: bytes, i: int) -> int:
        arr = (C.c_uint8 * 64).from_buffer_copy(block)
        return self.L.pho_clef_get(C.cast(arr, u8p), i)

    def load(self, ptrh: bytes) -> "PortIndex":
        return PortIndex(self, ptrh)


class PortIndex:
    def __init__(self, port: Port, ptrh: bytes):
        self.port = port
        self._buf = (C.c_uint8 * len(ptrh)).from_buffer_copy(ptrh)
        self.ix = PhoIndex()
        err = C.c_char_p()
        if port.L.pho_parse(C.cast(self._buf, u8p), len(ptrh), C.byref(self.ix), C.byref(err)):
            raise ValueError(err.value.decode())

    def __del__(self):
        try:
            self.port.L.pho_release(C.byref(self.ix))
        except Exception:
            pass

    def index(self, key: int, minimal=True) -> int:
        return self.port.L.pho_index_u64(C.byref(self.ix), key, int(minimal))

    def query_u64(self, keys, minimal=True):
        keys = np.ascontiguousarray(keys, dtype=np.uint64)
        out = np.empty(keys.size, dtype=np.uint64)
        self.port.L.pho_query_u64(C.byref(self.ix), _ptr(keys), keys.size, _ptr(out), int(minimal))
        return out

    def query_bytes(self, data, offsets, minimal=True):
        data = np.ascontiguousarray(data, dtype=np.uint8)
        offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        n = offsets.size - 1
        out = np.empty(n, dtype=np.uint64)
        self.port.L.pho_query_bytes(C.byref(self.ix), _ptr(data, u8p), _ptr(offsets), n,
                                    _ptr(out), int(minimal))
        return out


# ---- synthetic corpora (numpy; identical to corpus.hpp:14-16 / SURVEY §8d) ----
_GOLD = np.uint64(0x9E3779B97F4A7C15)


def mix64_np(z: np.ndarray) -> np.ndarray:
    z = z.copy()
    with np.errstate(over="ignore"):
        z ^= z >> np.uint64(30)
        z *= np.uint64(0xBF58476D1CE4E5B9)
        z ^= z >> np.uint64(27)
        z *= np.uint64(0x94D049BB133111EB)
        z ^= z >> np.uint64(31)
    return z


def corpus_u64_np(start: int, count: int, gen_seed: int) -> np.ndarray:
    i = np.arange(start + 1, start + count + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return mix64_np(np.uint64(gen_seed) + i * _GOLD)


def build_prepare_u64_np(keys: np.ndarray, P: int, S: int, seed: int):
    """Numpy restatement of one u64 build attempt's front phases (the oracle for
    ph_gpu_build_prepare_u64): hash_all H64{C*(key^seed)} (construction.cpp:98-111,
    hash.hpp:27); part = mul_hi(P, h) (engine.hpp:429) and the part-major arrangement with
    kOversubscribed when a part holds more than S keys (engine.hpp:412-474); each part sorted
    with kDuplicateHashes on equal neighbours (engine.hpp:505-518). part is monotone in h, so
    one global sort gives the part-major, per-part-sorted array."""
    k = np.ascontiguousarray(keys, dtype=np.uint64)
    with np.errstate(over="ignore"):
        h = np.sort(np.uint64(0x517CC1B727220A95) * (k ^ np.uint64(seed)))
        # mul_hi(P, h) for P < 2^32: (P*h_hi + (P*h_lo >> 32)) >> 32 without overflow
        part = (np.uint64(P) * (h >> np.uint64(32)) +
                ((np.uint64(P) * (h & np.uint64(0xFFFFFFFF))) >> np.uint64(32))) >> np.uint64(32)
    off = np.searchsorted(part, np.arange(P + 1, dtype=np.uint64), side="left").astype(np.uint64)
    if (np.diff(off) > S).any():
        return h, off, 1
    return h, off, 2 if (h.size > 1 and (h[1:] == h[:-1]).any()) else 0


def string_corpus(n: int, seed: int, lo=8, hi=64):
    """Small config-4 style string sets for tests: len U[lo,hi], bytes 0x21..0x7E, distinct."""
    import random
    r = random.Random(seed)
    seen, out = set(), []
    while len(out) < n:
        s = bytes(0x21 + r.randrange(94) for _ in range(lo + r.randrange(hi - lo + 1)))
        if s not in seen:
            seen.add(s)
            out.append(s)
    return out
