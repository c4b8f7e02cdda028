#!/usr/bin/env python
"""PtrHash query-path benchmark (BASELINE.json metric): batched MPHF query throughput in
Gkeys/s at n=1e9 u64 keys on one B200, with the pilot-gather / HBM roofline.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3] [--impl ours|reference]

A "step" is one pass of the query path over the config's whole query stream (config 3:
all 1e9 keys in a seeded shuffled order, u32 output, minimal with the CacheLineEF remap).

Our arm:
  * fixture (untimed): keys are generated, the index is built by the REFERENCE builder
    (oracle/_ref, as north_star requires — construction is not on the hot path), serialized
    to PTRH v1 and uploaded through the C ABI;
  * correctness gate (untimed): every GPU output is compared with the reference's own
    index_stream output, and the minimal outputs are checked to be a bijection on the GPU;
  * value: K device-timed steps (CUDA events on the launching stream; L2 flushed between
    steps outside the event pair; inputs 8 GB > L2 anyway), max over ranks;
  * e2e: K steps through the public host API (pinned host keys in, host u32 out; the
    library pipelines H2D -> kernel -> D2H), wall clock with syncs, max over ranks;
  * roofline: the query kernel's algorithmic bytes / its event-timed duration vs the
    measured HBM peak, plus the gather roofline of BASELINE.md §2 measured live;
  * cpu_baseline: the reference's index_stream(…, 32) on all host cores, on a bounded sample.
Reference arm (--impl reference): the reference's CPU query (index_stream, lookahead 32,
all host threads, contiguous slices as in the CLI bench) on a bounded sample per step.
"""
from __future__ import annotations

import argparse
import ctypes as C
import hashlib
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

GEN_SEED = 42          # corpus_u64 seed (CLI default gen_seed, ptrhash.cpp:234)
PERM_SEED = 7          # shuffled query order
SAMPLE_SEED = 0xC0FFEE  # config 2: sampling with replacement
METRIC = "batched MPHF query Gkeys/s (ns/key) at n=1e9 u64 keys; % of pilot-gather roofline"

CONFIGS = {
    1: dict(n=10**7, order="perm",
            desc="config1: n=1e7 distinct u64 (splitmix64), all keys in seeded shuffled order"),
    2: dict(n=10**8, order="sample",
            desc="config2: n=1e8 distinct u64, 1e8 queries sampled with replacement"),
    3: dict(n=10**9, order="perm",
            desc="config3: n=1e9 distinct u64 (8 GB keys, 333 MB pilots), all keys in seeded "
                 "shuffled order"),
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---------------------------------------------------------------------------
# distributed plumbing (one process per GPU; replicas, no data-path collective)
# ---------------------------------------------------------------------------
class Dist:
    def __init__(self, backend):
        import torch
        import torch.distributed as dist
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.dist = dist if self.world > 1 else None
        self.backend = backend
        if self.dist:
            if backend == "nccl":
                torch.cuda.set_device(self.local)
            dist.init_process_group(backend)

    def barrier(self):
        if self.dist:
            self.dist.barrier()

    def max(self, x: float) -> float:
        if not self.dist:
            return x
        import torch
        dev = "cuda" if self.backend == "nccl" else "cpu"
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.dist:
            self.dist.destroy_process_group()


# ---------------------------------------------------------------------------
# clocks during the timed region (NVML; the recipe's clocks line)
# ---------------------------------------------------------------------------
REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
           0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks",
           0x10: "sync_boost", 0x1: "gpu_idle"}


class ClockSampler:
    def __init__(self, device_index: int):
        self.samples = []
        self.windows = []
        self._stop = threading.Event()
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover
            log("clock sampler unavailable:", e)
            self.nv = None
        self.t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                util = nv.nvmlDeviceGetUtilizationRates(self.h).gpu
                self.samples.append((time.perf_counter(), sm, rs, util))
            except Exception:
                pass
            time.sleep(0.01)

    def start(self):
        if self.nv:
            self.t.start()

    def window(self, t0, t1):
        self.windows.append((t0, t1))

    def stop(self):
        self._stop.set()
        if self.nv:
            self.t.join(timeout=1)

    def summary(self):
        inside = [s for s in self.samples if any(a <= s[0] <= b for a, b in self.windows)]
        loaded = [s for s in inside if s[3] > 0] or inside
        if not loaded:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        bits = 0
        for s in loaded:
            bits |= s[2]
        reasons = sorted(name for b, name in REASONS.items() if bits & b and name != "gpu_idle")
        return {"sm_mhz": statistics.median(s[1] for s in loaded), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(loaded)}


# ---------------------------------------------------------------------------
# fixture: keys + reference-built index (untimed)
# ---------------------------------------------------------------------------
def ref_params(ref):
    # "default PtrHash parameters (λ=3.0, α=0.99, minimal with remap)": preset default
    # (cubic γ, CacheLineEF, fastmod) with λ = 3.0 (BASELINE.json configs)
    return ref.params("default", lambda_=(30, 10))


def build_index_bytes(n: int, dist: Dist, gen_keys) -> bytes:
    """Reference-built PTRH bytes; for N>1 rank 0 builds and shares through /dev/shm."""
    from oracle.bindings import Ref
    tag = hashlib.sha1(f"{n}-{GEN_SEED}-default-l30".encode()).hexdigest()[:12]
    shm = f"/dev/shm/ph_bench_{tag}_{os.getpid() if dist.world == 1 else 'job'}.ptrh"
    ptrh = None
    if dist.rank == 0:
        ref = Ref()
        t = time.time()
        keys = gen_keys(n)
        log(f"[fixture] {n} keys generated in {time.time() - t:.1f}s; building with the "
            f"reference builder ({ref.hw_threads()} threads)...")
        t = time.time()
        ptrh = ref.build_u64(keys, ref_params(ref), threads=0)
        log(f"[fixture] reference build {time.time() - t:.1f}s, PTRH {len(ptrh) / 1e6:.1f} MB")
        del keys
        if dist.world > 1:
            with open(shm, "wb") as f:
                f.write(ptrh)
    dist.barrier()
    if ptrh is None:
        with open(shm, "rb") as f:
            ptrh = f.read()
    dist.barrier()
    if dist.rank == 0 and dist.world > 1:
        os.unlink(shm)
    return ptrh


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args, cfg):
    import torch
    dist = Dist("nccl")
    torch.cuda.set_device(dist.local)
    from paper_2502_15539_b200 import ph_gpu
    bench = C.CDLL(os.path.join(ROOT, "paper_2502_15539_b200", "libph_bench.so"))
    n = cfg["n"]
    stream = torch.cuda.current_stream()
    sp = C.c_void_p(stream.cuda_stream)

    def gen_keys_gpu(count):
        keys = np.empty(count, dtype=np.uint64)
        chunk = 1 << 27
        buf = torch.empty(min(chunk, count), dtype=torch.int64, device="cuda")
        for s in range(0, count, chunk):
            m = min(chunk, count - s)
            assert bench.phb_gen_corpus(C.c_void_p(buf.data_ptr()), C.c_uint64(s), C.c_uint64(m),
                                        C.c_uint64(GEN_SEED), sp) == 0
            keys[s:s + m] = buf[:m].cpu().numpy().view(np.uint64)
        del buf
        return keys

    ptrh = build_index_bytes(n, dist, gen_keys_gpu)
    idx = ph_gpu.PtrHashIndex(ptrh, device=dist.local)
    info = idx.info
    nq = n  # queries per step per rank
    q = torch.empty(nq, dtype=torch.int64, device="cuda")
    seed = PERM_SEED + dist.rank if cfg["order"] == "perm" else SAMPLE_SEED + dist.rank
    fn = bench.phb_gen_queries_perm if cfg["order"] == "perm" else bench.phb_gen_queries_sample
    assert fn(C.c_void_p(q.data_ptr()), C.c_uint64(0), C.c_uint64(nq), C.c_uint64(n),
              C.c_uint64(GEN_SEED), C.c_uint64(seed), sp) == 0
    out = torch.empty(nq, dtype=torch.int32, device="cuda")
    out_nm = torch.empty(nq, dtype=torch.int32, device="cuda")

    # ---- correctness gate (untimed) ----
    idx.query(q, out=out, minimal=True, out_width=4)
    idx.query(q, out=out_nm, minimal=False, out_width=4)
    torch.cuda.synchronize()
    remap_frac = float((out_nm.to(torch.int64) & 0xFFFFFFFF).ge(n).double().mean().item())
    gate = {"remap_fraction": remap_frac}
    if cfg["order"] == "perm":
        bits = torch.zeros((n + 31) // 32, dtype=torch.int32, device="cuda")
        bad = torch.zeros(2, dtype=torch.int64, device="cuda")
        bench.phb_bijection(C.c_void_p(out.data_ptr()), C.c_uint64(nq), C.c_uint64(n),
                            C.c_void_p(bits.data_ptr()), C.c_void_p(bad.data_ptr()), sp)
        torch.cuda.synchronize()
        gate["bijection"] = bad.tolist() == [0, 0]
        del bits
    pin_q = torch.empty(nq, dtype=torch.int64).pin_memory()
    pin_q.copy_(q)
    pin_o = torch.empty(nq, dtype=torch.int32).pin_memory()
    if args.verify != "none" and dist.rank == 0:
        from oracle.bindings import Ref
        ref = Ref()
        ri = ref.load(ptrh)
        qh = pin_q.numpy().view(np.uint64)
        m = nq if args.verify == "full" else min(nq, 10**7)
        t = time.time()
        ok = True
        for minimal, o in ((True, out), (False, out_nm)):
            want = ri.query_u64(qh[:m], minimal, "stream", 32, threads=os.cpu_count() or 1)
            got = o[:m].cpu().numpy().view(np.uint32)
            ok &= bool(np.array_equal(got, want.astype(np.uint32))) and int(want.max()) < 2**32
            del want
        gate["bit_exact_vs_reference"] = ok
        gate["verified_queries"] = int(m) * 2
        log(f"[gate] {m} queries x (minimal, non-minimal) vs reference index_stream: "
            f"{'OK' if ok else 'MISMATCH'} ({time.time() - t:.1f}s)")
        ri.close()
        if not ok or not gate.get("bijection", True):
            raise SystemExit("correctness gate failed: " + json.dumps(gate))

    # ---- gather / HBM roofline microbenchmarks (live, same box) ----
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    def time_ms(fn_, reps=3):
        best = 1e30
        for _ in range(reps):
            flush.zero_()
            a, b = ev(), ev()
            a.record(stream)
            fn_()
            b.record(stream)
            b.synchronize()
            best = min(best, a.elapsed_time(b))
        return best

    src = torch.empty(1 << 31, dtype=torch.uint8, device="cuda")
    dst = torch.empty_like(src)
    copy_ms = time_ms(lambda: dst.copy_(src), 5)
    bw_copy = 2 * src.numel() / copy_ms / 1e6  # GB/s, read+write (MEASURED_PEAKS method)
    del src, dst
    pil = torch.empty(int(info.pilot_bytes), dtype=torch.uint8, device="cuda")
    sink = torch.zeros(1, dtype=torch.int32, device="cuda")
    nl = 1 << 28
    g_ms = time_ms(lambda: bench.phb_gather(C.c_void_p(pil.data_ptr()), C.c_uint64(pil.numel()),
                                            C.c_uint64(nl), C.c_uint64(1), 8, 8,
                                            C.c_void_p(sink.data_ptr()), sp))
    r_gather = nl / g_ms / 1e6  # G sectors/s
    del pil

    # ---- timed region: value ----
    sampler = ClockSampler(torch.cuda.current_device())
    sampler.start()

    def step(minimal=True):
        idx.query(q, out=out, minimal=minimal, out_width=4, stream=stream.cuda_stream)

    def timed(minimal):
        for _ in range(args.warmup):
            step(minimal)
        torch.cuda.synchronize()
        dist.barrier()
        torch.cuda.synchronize()
        l0 = ph_gpu.launch_count()
        t0 = time.perf_counter()
        ms = []
        for _ in range(args.steps):
            flush.zero_()  # L2 flush outside the event pair
            a, b = ev(), ev()
            a.record(stream)
            step(minimal)
            b.record(stream)
            ms.append((a, b))
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        dist.barrier()
        sampler.window(t0, t1)
        ms = [a.elapsed_time(b) for a, b in ms]
        return ms, ph_gpu.launch_count() - l0

    ms_min, launches = timed(True)
    ms_nm, _ = timed(False)
    total_ms = dist.max(sum(ms_min))
    total_nm = dist.max(sum(ms_nm))

    # ---- timed region: e2e through the public host API ----
    for _ in range(max(1, min(args.warmup, 2))):
        idx.query(pin_q, out=pin_o, minimal=True, out_width=4)
    dist.barrier()
    torch.cuda.synchronize()
    l0 = ph_gpu.launch_count()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        idx.query(pin_q, out=pin_o, minimal=True, out_width=4)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    e2e_launches = ph_gpu.launch_count() - l0
    dist.barrier()
    sampler.window(t0, t1)
    e2e_s = dist.max(t1 - t0)
    sampler.stop()
    step(True)  # the e2e outputs must equal the device-resident path's
    torch.cuda.synchronize()
    if not torch.equal(pin_o.cuda(), out):
        raise SystemExit("e2e host-path output differs from the device path")

    # ---- report ----
    N = dist.world
    K = args.steps
    value = N * nq * K / (total_ms * 1e-3) / 1e9
    kern_ms = statistics.mean(ms_min)
    sectors = 1.0 + remap_frac * (1.0 + 32.0 / 44.0)  # pilot + CLEF (i>=12 touches 2nd sector)
    bytes_per_key = 12.0 + 32.0 * sectors
    peak, peak_src = measured_peaks()
    achieved = nq * bytes_per_key / (kern_ms * 1e-3) / 1e9
    stream_ms = nq * 12.0 / (bw_copy * 1e9) * 1e3
    gather_ms = nq * sectors / (r_gather * 1e9) * 1e3
    t_roof = max(stream_ms, gather_ms)
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                tr = json.load(f)
            traffic = tr.get(f"config{args.config}", {}).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    cpu = None
    if dist.rank == 0 and N == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(ptrh, pin_q.numpy().view(np.uint64), args)
    res = {
        "metric": METRIC,
        "value": round(value, 3),
        "unit": "Gkeys/s",
        "ns_per_key": round(1.0 / value, 5),
        "n_gpus": N,
        "steps": K,
        "warmup": args.warmup,
        "ms_per_step": round(total_ms / K, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u64",
        "data": "synthetic (splitmix64 corpus_u64 keys, seeded Feistel shuffle; index built by "
                "the reference builder)",
        "config": {"workload": cfg["desc"], "n": n, "queries_per_step_per_gpu": nq,
                   "params": "preset default, lambda=3.0, alpha=0.99, cubic gamma, CacheLineEF, "
                             "fastmod S", "P": int(info.parts), "S": int(info.slots_per_part),
                   "B": int(info.buckets_per_part), "output": "u32, minimal",
                   "parallelism": f"replicas x{N} (no collective)",
                   "l2": "flushed between steps (512 MiB write, outside the timed events); "
                         "inputs (8 B/key) and pilots exceed L2 at n=1e9"},
        "nonminimal": {"value": round(N * nq * K / (total_nm * 1e-3) / 1e9, 3), "unit": "Gkeys/s",
                       "ms_per_step": round(total_nm / K, 4)},
        "gpu_launches": int(launches),
        "e2e": {"value": round(N * nq * K / e2e_s / 1e9, 4), "unit": "Gkeys/s",
                "h2d_bytes_per_step": nq * 8, "d2h_bytes_per_step": nq * 4,
                "api": "ph_gpu_index_stream_u64 (host pinned keys -> host u32 out)",
                "gpu_launches": int(e2e_launches)},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                     "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": traffic,
                     "peak_source": peak_src,
                     "algorithmic_bytes_per_key": round(bytes_per_key, 3),
                     "note": "12 B streamed (8 B key + 4 B out) + 32 B x (1 pilot sector + "
                             "remap_fraction x 1.727 CacheLineEF sectors)"},
        "gather_roofline": {"t_roof_ms": round(t_roof, 4), "t_measured_ms": round(kern_ms, 4),
                            "frac": round(t_roof / kern_ms, 4),
                            "stream_bound_ms": round(stream_ms, 4),
                            "gather_bound_ms": round(gather_ms, 4),
                            "copy_gbs": round(bw_copy, 1),
                            "r_gather_gsectors_s": round(r_gather, 3),
                            "gather_buffer_bytes": int(info.pilot_bytes)},
        "gate": gate,
        "clocks": sampler.summary(),
        "cpu_baseline": cpu,
    }
    if dist.rank == 0:
        print(json.dumps(res), flush=True)
    dist.close()


def cpu_baseline(ptrh: bytes, queries: np.ndarray, args):
    """The reference's index_stream(keys, 32, out, minimal) on all host cores, contiguous
    slices (proj/tools/ptrhash.cpp:486-512), one warm-up then best of 3 (:212-223)."""
    from oracle.bindings import Ref
    ref = Ref()
    ri = ref.load(ptrh)
    T = os.cpu_count() or 1
    S = min(queries.size, args.cpu_sample)
    sample = np.ascontiguousarray(queries[:S])
    out = np.empty(S, dtype=np.uint64)
    ri.query_u64(sample, True, "stream", 32, threads=T, out=out)
    best = 1e30
    for _ in range(3):
        t = time.perf_counter()
        ri.query_u64(sample, True, "stream", 32, threads=T, out=out)
        best = min(best, time.perf_counter() - t)
    ri.close()
    return {"value": round(S / best / 1e9, 4), "unit": "Gkeys/s", "ns_per_key": round(best / S * 1e9, 3),
            "cores": T, "kind": "reference",
            "sample": f"first {S} queries of the same shuffled stream, index_stream lookahead 32, "
                      f"minimal, {T} threads, best of 3 after 1 warm-up"}


# ---------------------------------------------------------------------------
# reference arm
# ---------------------------------------------------------------------------
def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle.bindings import Port, Ref
    n = cfg["n"]
    ref, port = Ref(), Port()
    T = os.cpu_count() or 1
    t = time.time()
    keys = port.gen_keys("corpus", 0, n, n, GEN_SEED)
    ptrh = ref.build_u64(keys, ref_params(ref), threads=0)
    del keys
    log(f"[reference] index built in {time.time() - t:.1f}s")
    ri = ref.load(ptrh)
    S = min(n, args.cpu_sample)
    kind = "perm" if cfg["order"] == "perm" else "sample"
    q = port.gen_keys(kind, 0, S, n, GEN_SEED, PERM_SEED if kind == "perm" else SAMPLE_SEED)
    out = np.empty(S, dtype=np.uint64)
    for _ in range(args.warmup):
        ri.query_u64(q, True, "stream", 32, threads=T, out=out)
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        ri.query_u64(q, True, "stream", 32, threads=T, out=out)
        ts.append(time.perf_counter() - t0)
    total = sum(ts)
    value = S * args.steps / total / 1e9
    sample = (f"first {S} queries of the config's query stream per step; reference "
              f"PtrHashIndex::index_stream(lookahead 32), minimal, {T} threads, contiguous slices")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(value, 5), "unit": "Gkeys/s",
        "ns_per_key": round(1 / value, 4), "n_gpus": int(os.environ.get("WORLD_SIZE", "1")),
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(total / args.steps * 1e3, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic", "config": {"workload": cfg["desc"], "n": n,
                                        "params": "preset default, lambda=3.0"},
        "cpu_baseline": {"value": round(value, 5), "unit": "Gkeys/s", "cores": T,
                         "kind": "reference", "sample": sample},
        "e2e": {"value": round(value, 5), "unit": "Gkeys/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=3, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--verify", default="full", choices=["full", "sample", "none"])
    ap.add_argument("--cpu-sample", type=int, default=100_000_000)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        log("note: warmup raised to 3 (timing rules)")
        args.warmup = 3
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
