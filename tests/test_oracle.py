"""CPU tests: pin the oracle (our plain-C restatement, oracle/ph_oracle.c) against the
reference's golden vectors (tests/golden/, made by the reference library) and against
the compiled reference itself (oracle/_ref/libptrhash_ref.so).

Mirrors the reference's primitive tests: test_hash.cpp:15-157, test_bucket_fn.cpp:15-137,
test_cacheline_ef.cpp:12-133, test_serde.cpp:72-132, test_query.cpp:23-74.
"""
import os
import random

import numpy as np
import pytest

from conftest import golden_names, load_golden

MASK = (1 << 64) - 1


# ---- known answers (regenerated from the reference) ----

def test_appendix_b_values(port):
    L = port.L
    S = 0x9E3779B97F4A7C15
    assert L.pho_hash_int(0x0123456789ABCDEF, S) == 0x5FFD03373B845A82
    assert L.pho_hash_pilot(255, S) == 0x5FD60E223C4FD832
    assert L.pho_reduce(761766, 0xFEDCBA9876543210) == 658998
    assert L.pho_reduce(1 << 20, 0xFEDCBA9876543210) == 380184
    x = 0xFEDCBA9876543210
    assert L.pho_gamma(1, x) == 0xFDBAC097C8DC5ACC
    assert L.pho_gamma(2, x) == 0xFD2C1AE06275DE4D
    assert L.pho_gamma(3, x) == 0xFE02468ACF13579C
    assert L.pho_gamma(4, x) == 0xF8B95684C2668321
    assert L.pho_gamma(2, 1 << 63) == 773 << 52  # test_bucket_fn.cpp:15-35
    assert L.pho_gamma(4, 1 << 63) == 0x279FAD1013012C00
    assert L.pho_gamma(1, 1 << 63) == 1 << 62
    assert port.hash_bytes(b"hello world", S, 1)[0] == 0xC77469177148303B
    assert port.hash_bytes(b"hello world", S, 3)[0] == 0x7DD9F99674EEBC1F
    assert port.hash_bytes(b"hello world", S, 2) == (0x2845EFDDD8F1F2BD, 0xD1FB928539F53CEE)
    assert port.hash_bytes(b"hello world", S, 4) == (0x34FE348ABDB118F8, 0xD4620988B36D2DA2)
    assert port.hash_bytes(b"", S, 1)[0] == 0x2F212123BA830CB9
    assert port.hash_bytes(b"", S, 3)[0] == 0xECB75C90701AB2F9
    assert port.hash_bytes(b"0123456789abcdef", S, 1)[0] == 0x06E9238CD9B11667
    assert port.hash_bytes(b"0123456789abcdefX", S, 1)[0] == 0x0A00BED2C279DFD3


def test_kat_primitives(port, kat):
    L = port.L
    for x, s, h in kat["hash_int"]:
        assert L.pho_hash_int(x, s) == h
    for p, s, h in kat["hash_pilot"]:
        assert L.pho_hash_pilot(p, s) == h
    for s, x, r in kat["reduce"]:
        assert L.pho_reduce(s, x) == r, (s, x)
        assert r < s
    for s, hi, lo in kat["fastmod_magic"]:
        assert port.fastmod_magic(s) == (hi, lo)
    for g, x, v in kat["gamma"]:
        assert L.pho_gamma(g, x) == v, (g, x)
    for h, P, B, g, part, bucket in kat["part_and_bucket"]:
        assert port.part_and_bucket(h, P, B, g) == (part, bucket)


def test_kat_string_hashes(port, kat):
    for s_hex, seed, algo, hi, lo in kat["hash_bytes"]:
        assert port.hash_bytes(bytes.fromhex(s_hex), seed, algo) == (hi, lo), (s_hex, seed, algo)


def test_kat_cacheline_ef(port, kat):
    for rec in kat["clef"]:
        if rec["status"] != 0:
            continue
        blk = bytes.fromhex(rec["block"])
        # pinned byte layout, cacheline_ef.hpp:58-73
        assert int.from_bytes(blk[0:4], "little") == rec["values"][0] >> 8
        for i, v in enumerate(rec["get"]):
            assert v == rec["values"][i]
            assert port.clef_get(blk, i) == v


def test_fastmod_matches_division(port):
    # test_hash.cpp:144-157: fastmod == 128-bit % for S in {3, 1000, 2^31-1} and boundaries
    rng = random.Random(1)
    for S in (3, 1000, (1 << 31) - 1, 761766, (1 << 32) - 1):
        xs = [0, 1, S - 1, S, S + 1, MASK, MASK - 1] + [rng.getrandbits(64) for _ in range(20000)]
        for x in xs:
            assert port.L.pho_reduce(S, x) == x % S


def test_cubic_matches_exact_rational(port):
    # test_bucket_fn.cpp:37-45 vs oracles.hpp:64-70 gamma3_exact
    rng = random.Random(2)
    for _ in range(20000):
        x = rng.getrandbits(64)
        x2 = (x * x) >> 64
        x3 = (x2 * x) >> 64
        half = (x2 + x3) >> 1
        assert port.L.pho_gamma(2, x) == ((half * 255) >> 8) + (x >> 8)


def test_gammas_monotone(port):
    # test_bucket_fn.cpp:47-66
    xs = sorted(random.Random(3).getrandbits(64) for _ in range(5000))
    for g in range(5):
        ys = [port.L.pho_gamma(g, x) for x in xs]
        assert all(a <= b for a, b in zip(ys, ys[1:])), g


def test_port_vs_reference_random_primitives(port, ref):
    rng = random.Random(4)
    for _ in range(3000):
        x, s = rng.getrandbits(64), rng.getrandbits(64)
        assert port.L.pho_hash_int(x, s) == ref.L.ref_hash_int(x, s)
        g = rng.randrange(5)
        assert port.L.pho_gamma(g, x) == ref.L.ref_gamma(g, x)
        S = rng.choice([rng.randrange(1, 1 << 32), 1 << rng.randrange(0, 40)])
        assert port.L.pho_reduce(S, x) == ref.L.ref_reduce(S, x)
    for _ in range(3000):
        b = bytes(rng.randrange(256) for _ in range(rng.randrange(0, 100)))
        seed = rng.getrandbits(64)
        for algo in range(5):
            assert port.hash_bytes(b, seed, algo) == ref.hash_bytes(b, seed, algo)


# ---- whole-index golden fixtures ----

@pytest.mark.parametrize("name", golden_names())
def test_port_matches_golden_index(port, name):
    from oracle.bindings import corpus_u64_np  # noqa: F401
    ptrh, rec = load_golden(name)
    pi = port.load(ptrh)
    if "queries" in rec:
        q = np.array(rec["queries"], dtype=np.uint64)
        assert pi.query_u64(q, True).tolist() == rec["minimal"]
        assert pi.query_u64(q, False).tolist() == rec["nonminimal"]
    else:
        strs = [bytes.fromhex(h) for h in rec["queries_hex"]]
        offs = np.zeros(len(strs) + 1, dtype=np.uint64)
        offs[1:] = np.cumsum([len(s) for s in strs])
        data = np.frombuffer(b"".join(strs), dtype=np.uint8)
        assert pi.query_bytes(data, offs, True).tolist() == rec["minimal"]
        assert pi.query_bytes(data, offs, False).tolist() == rec["nonminimal"]


def test_golden_member_queries_are_bijective(port):
    for name in golden_names():
        ptrh, rec = load_golden(name)
        n = int.from_bytes(ptrh[16:24], "little")
        if name.startswith("str_") and name != "str_default":
            continue  # hash id rewritten: arithmetic pinned, no longer a bijection
        assert sorted(rec["minimal"][:n]) == list(range(n)), name


# ---- parse / reject, test_serde.cpp:72-106 ----

def _corrupt_cases(ptrh: bytes):
    b = bytearray(ptrh)
    yield "magic", bytes(b"XTRH" + b[4:])
    v = bytearray(b); v[4] = 2
    yield "version", bytes(v)
    for off, name in ((8, "key kind"), (9, "hash"), (10, "bucket fn"), (11, "remap"), (12, "reduce")):
        c = bytearray(b); c[off] = 9
        yield name, bytes(c)
    yield "truncated", bytes(b[:-1])
    yield "trailing", bytes(b + b"\0")
    yield "header only", bytes(b[:40])
    z = bytearray(b); z[16:24] = (0).to_bytes(8, "little")
    yield "n=0", bytes(z)
    big = bytearray(b); big[16:24] = (1 << 40).to_bytes(8, "little")
    yield "n>slots", bytes(big)
    pl = bytearray(b); pl[56:64] = (int.from_bytes(b[56:64], "little") + 1).to_bytes(8, "little")
    yield "pilot len", bytes(pl)


def test_port_rejects_corrupt(port):
    ptrh, _ = load_golden("default_l30")
    port.load(ptrh)
    for what, bad in _corrupt_cases(ptrh):
        with pytest.raises(ValueError):
            port.load(bad)


def test_reference_rejects_same_corrupt(ref):
    ptrh, _ = load_golden("default_l30")
    for what, bad in _corrupt_cases(ptrh):
        with pytest.raises(ValueError):
            ref.load(bad)


# ---- the oracle on freshly built indexes vs the reference query (test_query.cpp:23-74) ----

@pytest.mark.parametrize("preset,over", [
    ("default", {"lambda_": (30, 10)}), ("fast", {}), ("compact", {}),
    ("default", {"remap": "elias-fano"}), ("default", {"bucket_fn": "optimal"}),
    ("default", {"bucket_fn": "skewed", "reduce": "pow2-mul"}),
])
def test_port_vs_reference_fresh_index(ref, port, preset, over):
    from oracle.bindings import corpus_u64_np
    n = 50_000
    keys = corpus_u64_np(0, n, 11)
    ptrh = ref.build_u64(keys, ref.params(preset, **over))
    ri, pi = ref.load(ptrh), port.load(ptrh)
    q = np.concatenate([keys, corpus_u64_np(0, n, 12)])
    for minimal in (True, False):
        want = ri.query_u64(q, minimal, "loop")
        assert np.array_equal(pi.query_u64(q, minimal), want)
        assert np.array_equal(ri.query_u64(q, minimal, "stream", 32), want)
        assert np.array_equal(ri.query_u64(q, minimal, "batched", 64, threads=3), want)
    out = pi.query_u64(keys, True)
    assert np.array_equal(np.sort(out), np.arange(n, dtype=np.uint64))
    assert pi.query_u64(q, True).max() < n  # non-members land below n too


def test_feistel_is_a_permutation(port):
    for n in (1, 2, 3, 1000, 4097, 65536):
        p = [port.L.pho_feistel_perm(i, n, 7) for i in range(n)]
        assert sorted(p) == list(range(n))


def test_kmer_oracle_matches_numpy(port):
    n_bases = 5_003
    seq = port.gen_dna(n_bases, 44)
    bases = np.array([(int(seq[j // 32]) >> (2 * (31 - j % 32))) & 3 for j in range(n_bases)])
    for k in (1, 5, 31, 32):
        want = []
        for i in range(0, n_bases - k + 1, 97):
            v = 0
            for t in range(k):
                v = (v << 2) | int(bases[i + t])
            want.append(v)
        got = port.kmers(seq, n_bases, k)[::97]
        assert [int(x) for x in got] == want
