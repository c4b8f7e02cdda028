"""Checked-build run of the partitioned path (compute-sanitizer is closed on this GPU pool).

Loads paper_2502_15539_b200/variants/libph_gpu_checked.so (built with -DPH_CHECKS: device-side
bounds checks on every shared-memory staging index, bulk-copy range and scatter position of
passes A-C, plus a canary band after the scratch), and for each case:
  * compares the outputs with the reference library (bit-exact),
  * reads the device check counters (ph_gpu_check_errors) -- must be 0,
  * repeats the call under different CTA counts per SM for passes A/B/C and compares the
    outputs: a race between the bulk copies, the mbarriers and the threads would show up as a
    difference between launch shapes or repeats.
Cases: u64 batches of 1, 4095..4097, 1e6+3 keys; unaligned key / output pointers; a single
key repeated (the spill region); keys sorted by group; many groups (small slices); k-mer
sources at the tile-edge sizes; u32 and u64 outputs; minimal and non-minimal; and builds
(u64 and string keys) with the GPU pilot search, whose kernel carries its own assertions.

  python tools/checked_run.py   (PH_GPU_LIB defaults to variants/libph_gpu_checked.so)
"""
import ctypes as C
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("PH_GPU_LIB", os.path.join(ROOT, "paper_2502_15539_b200", "variants",
                                                 "libph_gpu_checked.so"))

SHAPES = [("A2_B4_C3", {"PH_GPU_PART_A_CTAS": "2", "PH_GPU_PART_B_CTAS": "4", "PH_GPU_PART_C_CTAS": "3"}),
          ("A1_B1_C1", {"PH_GPU_PART_A_CTAS": "1", "PH_GPU_PART_B_CTAS": "1", "PH_GPU_PART_C_CTAS": "1"}),
          ("A2_B2_C2", {"PH_GPU_PART_A_CTAS": "2", "PH_GPU_PART_B_CTAS": "2", "PH_GPU_PART_C_CTAS": "2"})]


def main():
    import torch
    from oracle.bindings import Port, Ref, corpus_u64_np
    from paper_2502_15539_b200 import ph_gpu
    L = ph_gpu._L
    L.ph_gpu_check_errors.argtypes = [C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]

    def check_errors():
        c, line = C.c_uint64(), C.c_uint64()
        rc = L.ph_gpu_check_errors(C.byref(c), C.byref(line))
        assert rc == 0, f"not a checked build ({ph_gpu.LIB_PATH})"
        return int(c.value), int(line.value)

    ref, port = Ref(), Port()
    ph_gpu.set_partition(2)  # force the partitioned path on these small indexes
    results = []
    n = 200_000
    keys = corpus_u64_np(0, n, 42)
    ptrh = ref.build_u64(keys, ref.params("default", lambda_=(30, 10)))
    ri = ref.load(ptrh)
    idx = ph_gpu.PtrHashIndex(ptrh)

    def run_case(name, q_np, width=4, koff=0, ooff=0):
        q = np.ascontiguousarray(q_np, dtype=np.uint64)
        for minimal in (True, False):
            want = ri.query_u64(q, minimal, "loop", threads=os.cpu_count() or 1)
            outs = []
            for shape, kv_env in SHAPES:
                for k, v in kv_env.items():
                    os.environ[k] = v
                for rep in range(2):
                    if koff:  # keys koff words in: 8-B but not 16-B aligned (non-bulk pass A)
                        buf = torch.zeros(q.size * 8 + 16, dtype=torch.uint8, device="cuda")
                        buf[8 * koff:8 * koff + q.size * 8].copy_(torch.from_numpy(q.view(np.uint8)))
                        kp = buf.data_ptr() + 8 * koff
                    else:
                        dk = torch.from_numpy(q.view(np.int64)).cuda()
                        kp = dk.data_ptr()
                    ob = torch.zeros(q.size * width + 16, dtype=torch.uint8, device="cuda")
                    op = ob.data_ptr() + ooff * width
                    rc = L.ph_gpu_query_u64(idx._h, C.c_void_p(kp), q.size, C.c_void_p(op), width,
                                            int(minimal), None)
                    assert rc == 0, ph_gpu._L.ph_gpu_last_error()
                    torch.cuda.synchronize()
                    got = ob[ooff * width:(ooff + q.size) * width].cpu().numpy().view(
                        np.uint32 if width == 4 else np.uint64).astype(np.uint64)
                    outs.append(got)
            errs = check_errors()
            same = all(np.array_equal(o, outs[0]) for o in outs)
            exact = np.array_equal(outs[0], want)
            results.append({"case": name, "minimal": minimal, "width": width, "keys": int(q.size),
                            "bit_exact": bool(exact), "identical_across_shapes_and_repeats": bool(same),
                            "check_violations": errs[0], "first_line": errs[1]})
            print(json.dumps(results[-1]), flush=True)
        for k in ("PH_GPU_PART_A_CTAS", "PH_GPU_PART_B_CTAS", "PH_GPU_PART_C_CTAS"):
            os.environ.pop(k, None)

    mixed = np.concatenate([keys, corpus_u64_np(0, 1_000_003 - n, 43)])
    for nq in (1, 4095, 4096, 4097, 1_000_003):
        run_case(f"u64 nq={nq}", mixed[:nq])
    run_case("u64 nq=1e6+3 out u64", mixed, width=8)
    run_case("u64 keys +8 B and u32 out +4 B (not 16-B aligned)", mixed[:300_017], koff=1, ooff=1)
    run_case("u64 out +8 B (not 16-B aligned)", mixed[:300_017], width=8, ooff=1)
    run_case("one key repeated (spill region)", np.full(500_001, keys[7], dtype=np.uint64))
    g = (((keys ^ np.uint64(0x9E3779B97F4A7C15)) * np.uint64(0x517CC1B727220A95)) >> np.uint64(32))
    run_case("keys sorted by hash (group order)", keys[np.argsort(g, kind="stable")])
    os.environ["PH_GPU_PART_SLICE_KB"] = "12"  # many small groups (G up to 64)
    run_case("many groups (12 KiB slices)", mixed)
    os.environ.pop("PH_GPU_PART_SLICE_KB")

    # k-mer source at the tile edges
    for n_bases, k in ((100, 31), (4096 + 30, 31), (130 * 32 + 31, 31), (1_000_000 + 30, 31),
                       (777_777, 16)):
        seq = port.gen_dna(n_bases, 44)
        km = port.kmers(seq, n_bases, k)  # the reference answers the materialised k-mers
        want_ptrh = ref.build_u64(np.unique(km), ref.params("default", lambda_=(30, 10)))
        kidx = ph_gpu.PtrHashIndex(want_ptrh)
        kri = ref.load(want_ptrh)
        dseq = torch.from_numpy(seq.view(np.int64)).cuda()
        for minimal in (True, False):
            want = kri.query_u64(km, minimal, "loop", threads=os.cpu_count() or 1)
            outs = []
            for shape, kv_env in SHAPES:
                for kk, v in kv_env.items():
                    os.environ[kk] = v
                for rep in range(2):
                    o = kidx.query_kmers(dseq, n_bases, k, minimal=minimal, out_width=4)
                    torch.cuda.synchronize()
                    outs.append(o.cpu().numpy().view(np.uint32).astype(np.uint64))
            errs = check_errors()
            results.append({"case": f"k-mers n_bases={n_bases} k={k}", "minimal": minimal,
                            "width": 4, "keys": int(km.size),
                            "bit_exact": bool(np.array_equal(outs[0], want)),
                            "identical_across_shapes_and_repeats": bool(all(np.array_equal(x, outs[0]) for x in outs)),
                            "check_violations": errs[0], "first_line": errs[1]})
            print(json.dumps(results[-1]), flush=True)
        for kk in ("PH_GPU_PART_A_CTAS", "PH_GPU_PART_B_CTAS", "PH_GPU_PART_C_CTAS"):
            os.environ.pop(kk, None)
        kidx.close()
    # construction: builds with the GPU pilot search forced, on the checked library (slots,
    # visiting indices, bucket ids, hash positions and heap sizes asserted on the device);
    # repeated builds must give the same bytes, equal to the reference's
    ph_gpu.set_partition(0)
    ph_gpu.set_build_search(2)
    from oracle.bindings import string_corpus
    build_cases = [("default l=3.0 n=300k", "default", dict(lambda_=(30, 10)), 300_000),
                   ("compact (evictions) n=300k", "compact", {}, 300_000),
                   ("fast pow2 n=150k", "fast", dict(reduce="pow2-mul"), 150_000),
                   ("optimal gamma, forced shape n=40k", "default",
                    dict(bucket_fn="optimal", shape=(3, 20_000, 3_000)), 40_000),
                   ("tiny n=7", "default", {}, 7)]
    for name, preset, kw, bn in build_cases:
        bk = corpus_u64_np(0, bn, 900 + bn)
        if "shape" in kw:
            want = ref.build_u64_shape(bk, ref.params(preset, **{k: v for k, v in kw.items() if k != "shape"}),
                                       *kw["shape"])
        else:
            want = ref.build_u64(bk, ref.params(preset, **kw))
        outs = [ph_gpu.build_u64(bk, ph_gpu.build_params(preset, **kw)) for _ in range(2)]
        errs = check_errors()
        results.append({"case": f"build u64: {name}", "minimal": None, "width": None, "keys": bn,
                        "bit_exact": bool(outs[0] == want),
                        "identical_across_shapes_and_repeats": bool(outs[0] == outs[1]),
                        "check_violations": errs[0], "first_line": errs[1]})
        print(json.dumps(results[-1]), flush=True)
    strs = string_corpus(80_000, 5) + [b"", b"x" * 300]
    so = np.zeros(len(strs) + 1, dtype=np.uint64)
    so[1:] = np.cumsum([len(x) for x in strs])
    sd = np.frombuffer(b"".join(strs), dtype=np.uint8).copy()
    want = ref.build_bytes(sd, so, ref.params("default"))
    outs = [ph_gpu.build_bytes(sd, so, ph_gpu.build_params("default")) for _ in range(2)]
    errs = check_errors()
    results.append({"case": "build strings (aes64) n=80k", "minimal": None, "width": None, "keys": len(strs),
                    "bit_exact": bool(outs[0] == want), "identical_across_shapes_and_repeats": bool(outs[0] == outs[1]),
                    "check_violations": errs[0], "first_line": errs[1]})
    print(json.dumps(results[-1]), flush=True)
    ph_gpu.set_build_search(0)
    ok = all(r["bit_exact"] and r["identical_across_shapes_and_repeats"] and r["check_violations"] == 0
             for r in results)
    print(f"CHECKED RUN {'CLEAN' if ok else 'FAILED'}: {len(results)} cases", flush=True)
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
