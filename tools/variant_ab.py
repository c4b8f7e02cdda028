"""A/B timing of library variants on a synthetic index of a config's shape (not the product,
not a parity test): each (library, environment) runs in its own process, times the whole
query call and each partitioned pass with CUDA events, and prints a hash of its outputs,
which must agree between variants (the parity tests check the values themselves).

  python tools/variant_ab.py --config 3 --runs "base:libph_gpu.so;nofb:variants/libph_gpu_nofb.so@PH_GPU_NO_MODFAST=1"

A run is NAME:LIB[@K=V,K=V]; LIB is relative to paper_2502_15539_b200/. --kmers times the
fused k-mer front end (config 5 shape) instead of u64 keys.
"""
import argparse
import hashlib
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def child(a):
    import torch
    from paper_2502_15539_b200 import ph_gpu
    from tools.synth_perf import SHAPES, synth_ptrh
    ptrh = synth_ptrh(a.config)
    if a.strings:  # the same shape as a string index hashed with aes64 (header bytes 8, 9)
        ptrh = ptrh[:8] + bytes([1, 1]) + ptrh[10:]
    idx = ph_gpu.PtrHashIndex(ptrh)
    idx.set_l2_policy(0, 2)  # file order, no window: DRAM-sized batches take the partitioned path
    n = a.nq or SHAPES[a.config][0]
    g = torch.Generator(device="cuda")
    g.manual_seed(7)
    if a.strings:  # config-4 strings (len U[8,64], bytes 0x21-0x7E), shuffled, device-generated
        import ctypes as C
        bench = C.CDLL(os.path.join(ROOT, "paper_2502_15539_b200", "libph_bench.so"))
        lens = torch.empty(n, dtype=torch.int64, device="cuda")
        assert bench.phb_str_lens(C.c_void_p(lens.data_ptr()), C.c_uint64(n), C.c_uint64(43),
                                  C.c_uint64(7), 1, None) == 0
        offs = torch.zeros(n + 1, dtype=torch.int64, device="cuda")
        torch.cumsum(lens, 0, out=offs[1:])
        del lens
        data = torch.empty(int(offs[-1].item()), dtype=torch.uint8, device="cuda")
        assert bench.phb_str_bytes(C.c_void_p(offs.data_ptr()), C.c_uint64(n), C.c_uint64(43),
                                   C.c_uint64(7), 1, C.c_void_p(data.data_ptr()), None) == 0
        torch.cuda.synchronize()
        run = lambda out, m: idx.query((data, offs), out=out, minimal=m, out_width=4)  # noqa
    elif a.kmers:
        nb = n + 30
        seq = torch.randint(-2**63, 2**63 - 1, ((nb + 31) // 32,), dtype=torch.int64,
                            device="cuda", generator=g)
        run = lambda out, m: idx.query_kmers(seq, nb, 31, out=out, minimal=m, out_width=4)  # noqa
    else:
        keys = torch.randint(-2**63, 2**63 - 1, (n,), dtype=torch.int64, device="cuda", generator=g)
        run = lambda out, m: idx.query(keys, out=out, minimal=m, out_width=4)  # noqa
    out = torch.empty(n, dtype=torch.int32, device="cuda")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    res = {}
    if a.ncu:  # one call per mode for the profiler, no timing
        for minimal in (True, False):
            run(out, minimal)
        torch.cuda.synchronize()
        print("RESULT {}", flush=True)
        return
    for minimal in (True, False):
        for _ in range(3):
            run(out, minimal)
        torch.cuda.synchronize()
        ts = []
        ph_gpu.set_pass_timing(True)
        for _ in range(a.reps):
            if a.gap_ms:  # idle gap between steps (power / clock headroom probe)
                torch.cuda.synchronize()
                time.sleep(a.gap_ms / 1e3)
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            run(out, minimal)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        sums, calls = ph_gpu.pass_times()
        ph_gpu.set_pass_timing(False)
        ts.sort()
        h = hashlib.sha1(out.cpu().numpy().tobytes()).hexdigest()[:16]
        res["min" if minimal else "nonmin"] = {
            "best_ms": round(ts[0], 4), "median_ms": round(ts[len(ts) // 2], 4),
            "passes_ms": [round(x / max(calls, 1), 4) for x in sums], "hash": h}
    print("RESULT " + json.dumps(res), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--runs", required=True)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--repeat", type=int, default=1, help="interleaved repetitions of the list")
    ap.add_argument("--kmers", action="store_true")
    ap.add_argument("--strings", action="store_true", help="config-4 strings on an aes64 index")
    ap.add_argument("--nq", type=int, default=0, help="queries (default: the shape's n)")
    ap.add_argument("--ncu", action="store_true", help="child only: one call per mode")
    ap.add_argument("--gap-ms", type=float, default=0.0, help="idle time between timed steps")
    ap.add_argument("--child", action="store_true")
    a = ap.parse_args()
    if a.child:
        return child(a)
    runs = [r for r in a.runs.split(";") if r]
    hashes = {}
    for rep in range(a.repeat):
        for r in runs:
            name, rest = r.split(":", 1)
            lib, _, kv = rest.partition("@")
            env = dict(os.environ)
            env["PH_GPU_LIB"] = os.path.join(ROOT, "paper_2502_15539_b200", lib)
            for item in filter(None, kv.split(",")):
                k, v = item.split("=", 1)
                env[k] = v
            cmd = [sys.executable, __file__, "--child", "--config", str(a.config), "--runs", "-",
                   "--reps", str(a.reps), "--nq", str(a.nq), "--gap-ms", str(a.gap_ms)] + (["--kmers"] if a.kmers else []) + \
                (["--strings"] if a.strings else [])
            p = subprocess.run(cmd, env=env, capture_output=True, text=True)
            line = [x for x in p.stdout.splitlines() if x.startswith("RESULT ")]
            if p.returncode or not line:
                print(f"{name}: FAILED rc={p.returncode}\n{p.stdout[-2000:]}\n{p.stderr[-3000:]}",
                      flush=True)
                continue
            d = json.loads(line[0][7:])
            for k, v in d.items():
                hashes.setdefault(k, set()).add(v["hash"])
                print(f"[{rep}] {name:14s} {k:6s} best {v['best_ms']:7.3f} median {v['median_ms']:7.3f} "
                      f"passes {v['passes_ms']}  out {v['hash']}", flush=True)
    for k, hs in hashes.items():
        print(f"{k}: outputs {'IDENTICAL' if len(hs) == 1 else 'DIFFER: ' + str(hs)}", flush=True)


if __name__ == "__main__":
    main()
