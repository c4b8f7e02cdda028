"""Generates the committed golden fixtures from the REFERENCE library itself.

Run in the build container (needs oracle/_ref/libptrhash_ref.so, i.e. `make -C oracle`):
    python tests/golden/gen_golden.py

Writes into tests/golden/:
  kat.json              known answers for the query-path primitives (hash_int, hash_pilot,
                        reduce/fastmod, the five gammas, part_and_bucket, string hashes for
                        all five algorithm ids, CacheLineEF encode/get) — every value computed
                        by the reference (SURVEY Appendix B lists a subset);
  idx_<name>.ptrh       small PTRH v1 indexes built by the reference builder, covering every
                        bucket function, remap encoding and reduce path, plus string indexes;
  idx_<name>.json       their queries (members + non-members) and the reference's index() /
                        index_no_remap() answers.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.bindings import Ref, corpus_u64_np, string_corpus  # noqa: E402

SEED = 0x9E3779B97F4A7C15
KAT_X = [0, 1, 2, 255, 256, 12345, 1 << 32, (1 << 63) - 1, 1 << 63, 0xFEDCBA9876543210,
         0x0123456789ABCDEF, (1 << 64) - 1, 0x8000000000000001, 0x5555555555555555]


def concat(strs):
    offs = np.zeros(len(strs) + 1, dtype=np.uint64)
    offs[1:] = np.cumsum([len(s) for s in strs])
    return np.frombuffer(b"".join(strs) or b"\0", dtype=np.uint8).copy(), offs


def kats(ref: Ref):
    L = ref.L
    k = {"seed": SEED, "C_inverse": L.ref_mix_constant_inverse()}
    k["hash_int"] = [[x, s, L.ref_hash_int(x, s)] for x in KAT_X for s in (0, SEED, 42)]
    k["hash_pilot"] = [[p, s, L.ref_hash_pilot(p, s)] for p in (0, 1, 7, 128, 255) for s in (0, SEED)]
    slots = [1, 2, 3, 1000, 1 << 20, 388501, 573922, 664541, 761766, (1 << 31) - 1, (1 << 32) - 1]
    k["reduce"] = [[s, x, L.ref_reduce(s, x)] for s in slots for x in KAT_X]
    k["fastmod_magic"] = [[s, *ref.fastmod_magic(s)] for s in slots if s & (s - 1)]
    k["gamma"] = [[g, x, L.ref_gamma(g, x)] for g in range(5) for x in KAT_X]
    k["part_and_bucket"] = [[h, P, B, g, *ref.part_and_bucket(h, P, B, g)]
                            for h in KAT_X for (P, B) in ((1, 5), (26, 128206), (1326, 251383))
                            for g in range(5)]
    strs = [b"", b"a", b"hello world", b"0123456789abcdef", b"0123456789abcdefX",
            b"x" * 31, b"y" * 32, b"z" * 33, bytes(range(64)), bytes(range(255, 175, -1))]
    k["hash_bytes"] = [[s.hex(), seed, algo, *ref.hash_bytes(s, seed, algo)]
                       for s in strs for seed in (SEED, 0, 7) for algo in range(5)]
    # CacheLineEF: encode a few value runs, record the 64 bytes and every get()
    rng = np.random.default_rng(5)
    clef = []
    for cnt, span in ((1, 0), (44, 0), (44, 21504), (20, 300), (44, 5000)):
        base = int(rng.integers(0, 1 << 30))
        vals = np.sort(base + rng.integers(0, span + 1, size=cnt)).astype(np.uint64)
        vals[-1] = vals[0] + span if cnt > 1 else vals[-1]
        vals = np.sort(vals)
        st, blk = ref.clef_encode(vals)
        clef.append({"values": [int(v) for v in vals], "status": st, "block": blk.hex(),
                     "get": [ref.clef_get(blk, i) for i in range(cnt)] if st == 0 else []})
    k["clef"] = clef
    return k


def write_index(ref, name, ptrh: bytes, queries, strings=None):
    with open(os.path.join(HERE, f"idx_{name}.ptrh"), "wb") as f:
        f.write(ptrh)
    ri = ref.load(ptrh)
    rec = {"name": name}
    if strings is None:
        q = np.asarray(queries, dtype=np.uint64)
        rec["queries"] = [int(x) for x in q]
        rec["minimal"] = [int(v) for v in ri.query_u64(q, True, "loop")]
        rec["nonminimal"] = [int(v) for v in ri.query_u64(q, False, "loop")]
    else:
        data, offs = concat(strings)
        rec["queries_hex"] = [s.hex() for s in strings]
        rec["minimal"] = [int(v) for v in ri.query_bytes(data, offs, True, "loop")]
        rec["nonminimal"] = [int(v) for v in ri.query_bytes(data, offs, False, "loop")]
    with open(os.path.join(HERE, f"idx_{name}.json"), "w") as f:
        json.dump(rec, f)
    ri.close()


def main():
    ref = Ref()
    with open(os.path.join(HERE, "kat.json"), "w") as f:
        json.dump(kats(ref), f, indent=0)

    n = 3000
    keys = corpus_u64_np(0, n, 42)
    nonmem = corpus_u64_np(0, n, 4242)
    queries = np.concatenate([keys, nonmem])
    cases = {
        "default_l30": ref.params("default", lambda_=(30, 10)),
        "fast": ref.params("fast"),
        "compact": ref.params("compact"),
        "quadratic_ef": ref.params("default", bucket_fn="quadratic", remap="elias-fano"),
        "skewed_plain": ref.params("default", bucket_fn="skewed", remap="plain32"),
        "optimal_clef": ref.params("default", bucket_fn="optimal"),
        "pow2_cubic": ref.params("default", reduce="pow2-mul"),
        "single_part": ref.params("default", reduce="fastmod-single", remap="plain32"),
        "alpha1_linear": ref.params("fast", alpha=(1, 1)),
    }
    for name, p in cases.items():
        write_index(ref, name, ref.build_u64(keys, p, threads=1), queries)
    # forced shapes from the reference's own tests (test_construction.cpp:277-320)
    one = np.array([12345], dtype=np.uint64)
    write_index(ref, "shape_one_slot", ref.build_u64_shape(one, ref.params("fast"), 1, 1, 1),
                np.concatenate([one, corpus_u64_np(0, 50, 8)]))
    k23 = corpus_u64_np(0, 23, 99)
    write_index(ref, "shape_2x16x5",
                ref.build_u64_shape(k23, ref.params("fast", retries=50), 2, 16, 5),
                np.concatenate([k23, corpus_u64_np(0, 50, 9)]))
    k500 = corpus_u64_np(0, 500, 5)
    write_index(ref, "shape_1x1024x5000",
                ref.build_u64_shape(k500, ref.params("fast"), 1, 1024, 5000),
                np.concatenate([k500, corpus_u64_np(0, 200, 10)]))
    # string keys: AES (this host has AES-NI) and portable
    strs = string_corpus(2000, 43)
    data, offs = concat(strs)
    extra = string_corpus(300, 44, 0, 80)
    ptrh = ref.build_bytes(data, offs, ref.params("default", lambda_=(30, 10)), threads=1)
    write_index(ref, "str_default", ptrh, None, strings=strs + extra)
    # The builder picks the string hash from the build host (hash.cpp:41-47: aes64 here).
    # To pin the other four ids, the header's hash-id byte (offset 9, serde.hpp:18) is
    # rewritten: the result is no longer a bijection, but the query arithmetic is fully
    # defined and the reference's answers are the parity target.
    for algo_name, algo in (("fx64", 0), ("aes128", 2), ("portable64", 3), ("portable128", 4)):
        patched = bytearray(ptrh)
        patched[9] = algo
        write_index(ref, f"str_{algo_name}", bytes(patched), None, strings=strs + extra)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
