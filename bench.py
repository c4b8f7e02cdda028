#!/usr/bin/env python
"""PtrHash query-path benchmark (BASELINE.json metric): batched MPHF query throughput in
Gkeys/s at n=1e9 u64 keys on one B200, with the pilot-gather / HBM roofline.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 1..5] [--impl ours|reference]

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

STR_SEED = 43          # config 4 string corpus
DNA_SEED = 44          # config 5 sequence

CONFIGS = {
    1: dict(kind="u64", n=10**7, order="perm",
            desc="config1: n=1e7 distinct u64 (splitmix64), all keys in seeded shuffled order"),
    2: dict(kind="u64", n=10**8, order="sample",
            desc="config2: n=1e8 distinct u64, 1e8 queries sampled with replacement"),
    3: dict(kind="u64", n=10**9, order="perm", layout="file",
            desc="config3: n=1e9 distinct u64 (8 GB keys, 333 MB pilots), all keys in seeded "
                 "shuffled order"),
    4: dict(kind="str", n=3 * 10**8, order="perm",
            desc="config4: n=3e8 distinct strings, len U[8,64], bytes 0x21-0x7E, one "
                 "concatenated buffer + u64 offsets, all keys in seeded shuffled order"),
    5: dict(kind="kmer", n=10**9, k=31, layout="file",
            desc="config5: every 31-mer of a seeded random ACGT sequence of 1e9+30 bases "
                 "(2-bit packed, first base in the MSBs), in sequence order; fused on-device "
                 "k-mer extraction"),
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
        capped = sum(1 for s in loaded if s[2] & 0x4)  # sw_power_cap bit
        return {"sm_mhz": statistics.median(s[1] for s in loaded), "sm_max_mhz": self.max_mhz,
                "sm_min_mhz": min(s[1] for s in loaded), "reasons": reasons, "samples": len(loaded),
                "sw_power_cap_share": round(capped / len(loaded), 3)}


# ---------------------------------------------------------------------------
# fixture: keys + reference-built index (untimed)
# ---------------------------------------------------------------------------
def ref_params(ref):
    # "default PtrHash parameters (λ=3.0, α=0.99, minimal with remap)": preset default
    # (cubic γ, CacheLineEF, fastmod) with λ = 3.0 (BASELINE.json configs)
    return ref.params("default", lambda_=(30, 10))


def build_index_bytes(n: int, dist: Dist, gen_keys, build=None, tag="u64", after=None) -> bytes:
    """Reference-built PTRH bytes; for N>1 rank 0 builds and shares through /dev/shm.
    gen_keys(n) -> u64 keys for the reference u64 builder, or build() -> PTRH bytes.
    after(keys, ptrh, ref_seconds, ref_threads) runs on rank 0 once the reference build is done
    (the construction comparison)."""
    from oracle.bindings import Ref
    tag = hashlib.sha1(f"{tag}-{n}-{GEN_SEED}-default-l30".encode()).hexdigest()[:12]
    shm = f"/dev/shm/ph_bench_{tag}_{os.getpid() if dist.world == 1 else 'job'}.ptrh"
    ptrh = None
    if dist.rank == 0:
        ref = Ref()
        t = time.time()
        if build is not None:
            ptrh = build()
        else:
            keys = gen_keys(n)
            log(f"[fixture] {n} keys generated in {time.time() - t:.1f}s; building with the "
                f"reference builder ({ref.hw_threads()} threads)...")
            t = time.time()
            ptrh = ref.build_u64(keys, ref_params(ref), threads=0)
            if after is not None:
                after(keys, ptrh, time.time() - t, ref.hw_threads())
            del keys
        log(f"[fixture] reference build {time.time() - t:.1f}s, PTRH {len(ptrh) / 1e6:.1f} MB")
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


def ptrh_shape(ptrh: bytes) -> dict:
    """n, P, S, B and the query-relevant ids from a PTRH v1 header (serde.hpp:12-31)."""
    import struct
    key_kind, algo, fn, remap, reduce_ = ptrh[8], ptrh[9], ptrh[10], ptrh[11], ptrh[12]
    n, P, S, B = struct.unpack_from("<QQQQ", ptrh, 16)
    return {"n": n, "P": P, "S": S, "B": B, "hash": algo, "bucket_fn": fn, "remap": remap,
            "key_kind": key_kind, "reduce": reduce_}


def config_dict(cfg: dict, ptrh: bytes, world: int) -> dict:
    """The workload as both arms print it (the driver compares the two `config`s)."""
    sh = ptrh_shape(ptrh)
    return {"workload": cfg["desc"], "n": sh["n"], "queries_per_step_per_gpu": cfg["nq"],
            "params": "preset default, lambda=3.0, alpha=0.99, cubic gamma, CacheLineEF, "
                      "fastmod S",
            "P": sh["P"], "S": sh["S"], "B": sh["B"], "hash": sh["hash"],
            "output": "u32, minimal", "parallelism": f"replicas x{world} (no collective)"}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


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
# ---------------------------------------------------------------------------
# workloads (our arm): index fixture, device-resident query, host-API query, gate
# ---------------------------------------------------------------------------
class U64Work:
    """configs 1-3: u64 keys, device-generated query stream (shuffled or sampled)."""

    stream_bytes = 12.0  # 8 B key in + 4 B u32 out

    def __init__(self, args, cfg, dist, bench, sp):
        import torch
        from paper_2502_15539_b200 import ph_gpu
        self.cfg, self.n = cfg, cfg["n"]
        n = self.n

        def gen_keys_gpu(count):
            keys = np.empty(count, dtype=np.uint64)
            chunk = 1 << 27
            buf = torch.empty(min(chunk, count), dtype=torch.int64, device="cuda")
            for s in range(0, count, chunk):
                m = min(chunk, count - s)
                assert bench.phb_gen_corpus(C.c_void_p(buf.data_ptr()), C.c_uint64(s),
                                            C.c_uint64(m), C.c_uint64(GEN_SEED), sp) == 0
                keys[s:s + m] = buf[:m].cpu().numpy().view(np.uint64)
            return keys

        self.construction = None

        def compare_build(keys, ptrh, ref_s, ref_threads):
            """Construction (off the query path): the same keys and parameters
            through ph_gpu_build_u64 (hash, sort and the per-part pilot search on the GPU),
            timed by wall clock like the reference build, and its PTRH bytes compared with the
            reference's."""
            if not args.construction or dist.world > 1:
                return
            gp = ph_gpu.build_params("default", lambda_=(30, 10))
            ph_gpu.build_u64(keys[:200_000], gp, threads=0, device=dist.local)  # untimed: loads the kernels
            t = time.time()
            ours, st = ph_gpu.build_u64(keys, gp, threads=0, device=dist.local, stats=True)
            ours_s = time.time() - t
            same = ours == ptrh
            log(f"[construction] reference {ref_s:.1f}s, ours {ours_s:.1f}s "
                f"(prepare {st['prepare_ms']:.0f} ms, search {st['search_ms']:.0f} ms), "
                f"PTRH identical: {same}")
            if not same:
                raise SystemExit("construction: ph_gpu_build_u64 bytes differ from the reference's")
            self.construction = {
                "what": "build(keys) + serialize() of this config's index from host-resident keys: "
                        "the reference's build() on all host threads vs ph_gpu_build_u64 "
                        "(hash + MSD radix sort + part offsets and the per-part pilot search on "
                        "the GPU, remap table on the host); wall clock, one run each, after one "
                        "untimed 2e5-key build that loads the kernels",
                "n": int(keys.size), "reference_s": round(ref_s, 3), "ours_s": round(ours_s, 3),
                "speedup": round(ref_s / ours_s, 3), "host_threads": int(ref_threads),
                "identical_ptrh": same, "attempts": st["attempts"],
                "search_on_gpu": bool(st.get("search_on_gpu")),
                "stages_ms": {k: round(st[k], 1) for k in
                              ("upload_ms", "prepare_ms", "search_ms", "remap_ms", "total_ms")}}

        self.ptrh = build_index_bytes(n, dist, gen_keys_gpu, after=compare_build)
        self.idx = ph_gpu.PtrHashIndex(self.ptrh, device=dist.local)
        if cfg.get("layout") == "file":
            # file-order pilots without a persisting window: device-resident batches of
            # this size then take the partitioned path (ph_gpu.h)
            self.idx.set_l2_policy(0, 2)
        elif cfg.get("layout") == "hot":
            self.idx.set_l2_policy(64 << 20, 0)  # hot-first + window: the direct kernel
        self.nq = n
        self.q = torch.empty(self.nq, dtype=torch.int64, device="cuda")
        perm = cfg["order"] == "perm"
        seed = (PERM_SEED if perm else SAMPLE_SEED) + dist.rank
        fn = bench.phb_gen_queries_perm if perm else bench.phb_gen_queries_sample
        assert fn(C.c_void_p(self.q.data_ptr()), C.c_uint64(0), C.c_uint64(self.nq), C.c_uint64(n),
                  C.c_uint64(GEN_SEED), C.c_uint64(seed), sp) == 0
        self.bijective = perm
        self.pin_q = torch.empty(self.nq, dtype=torch.int64).pin_memory()
        self.pin_q.copy_(self.q)
        self.h2d, self.d2h = self.nq * 8, self.nq * 4
        self.api = "ph_gpu_index_stream_u64 (host pinned u64 keys -> host u32 out)"

    def query(self, out, minimal, stream):
        self.idx.query(self.q, out=out, minimal=minimal, out_width=4, stream=stream)

    def e2e(self, pin_out):
        self.idx.query(self.pin_q, out=pin_out, minimal=True, out_width=4)

    def reference_answers(self, ri, minimal, m):
        qh = self.pin_q.numpy().view(np.uint64)[:m]
        return ri.query_u64(qh, minimal, "stream", 32, threads=os.cpu_count() or 1)

    def cpu_runner(self, ri, S):
        """run(count, minimal, mode, width, threads): the reference's bulk query over the
        first `count` queries of this stream (host copy, untimed)."""
        sample = np.ascontiguousarray(self.pin_q.numpy().view(np.uint64)[:S])
        out = np.empty(S, dtype=np.uint64)

        def run(count, minimal, mode, width, threads):
            ri.query_u64(sample[:count], minimal, mode, width, threads=threads, out=out[:count])
        return run, "queries of the same shuffled stream", lambda: None


class StrWork:
    """config 4: byte-string keys (concatenated bytes + u64 offsets), shuffled."""

    def __init__(self, args, cfg, dist, bench, sp):
        import torch
        from oracle.bindings import Ref
        from paper_2502_15539_b200 import ph_gpu
        self.cfg, self.n = cfg, cfg["n"]
        n = self.n

        def gen(permuted):
            lens = torch.empty(n, dtype=torch.int64, device="cuda")
            assert bench.phb_str_lens(C.c_void_p(lens.data_ptr()), C.c_uint64(n),
                                      C.c_uint64(STR_SEED), C.c_uint64(PERM_SEED + dist.rank),
                                      permuted, sp) == 0
            offs = torch.zeros(n + 1, dtype=torch.int64, device="cuda")
            torch.cumsum(lens, 0, out=offs[1:])
            del lens
            total = int(offs[-1].item())
            data = torch.empty(max(total, 1), dtype=torch.uint8, device="cuda")
            assert bench.phb_str_bytes(C.c_void_p(offs.data_ptr()), C.c_uint64(n),
                                       C.c_uint64(STR_SEED), C.c_uint64(PERM_SEED + dist.rank),
                                       permuted, C.c_void_p(data.data_ptr()), sp) == 0
            return data, offs

        def build():
            data, offs = gen(0)  # generation order, for the reference builder
            hd = data.cpu().numpy()
            ho = offs.cpu().numpy().view(np.uint64)
            del data, offs
            ref = Ref()
            log(f"[fixture] {n} strings ({hd.size / 1e9:.1f} GB) generated; reference "
                f"build_sharded over the concatenated buffer...")
            t = time.time()
            ptrh = ref.build_bytes(hd, ho, ref_params(ref), lean=True)
            ref_s = time.time() - t
            if args.construction and dist.world == 1 and ptrh[9] == 1:
                # Construction (off the query path): the same strings through ph_gpu_build_bytes
                # (string hash, sort and pilot search on the GPU), wall clock from host buffers
                gp = ph_gpu.build_params("default", lambda_=(30, 10))
                ph_gpu.build_bytes(hd[:int(ho[100_000])], ho[:100_001], gp)  # untimed: loads the kernels
                t = time.time()
                ours, st = ph_gpu.build_bytes(hd, ho, gp, hash_algo=1, stats=True)
                ours_s = time.time() - t
                same = ours == ptrh
                log(f"[construction] strings: reference {ref_s:.1f}s, ours {ours_s:.1f}s, PTRH identical: {same}")
                if not same:
                    raise SystemExit("construction: ph_gpu_build_bytes bytes differ from the reference's")
                self.construction = {
                    "what": "build(span<string>) + serialize() of this config's index from host-resident "
                            "bytes + offsets: the reference (build_sharded, one shard, all host threads) vs "
                            "ph_gpu_build_bytes (aes64 string hash, MSD radix sort and pilot search on the "
                            "GPU, remap table on the host); wall clock, one run each, after one untimed "
                            "1e5-key build that loads the kernels",
                    "n": int(n), "reference_s": round(ref_s, 3), "ours_s": round(ours_s, 3),
                    "speedup": round(ref_s / ours_s, 3), "host_threads": int(ref.hw_threads()),
                    "identical_ptrh": same, "attempts": st["attempts"],
                    "search_on_gpu": bool(st.get("search_on_gpu")),
                    "stages_ms": {k: round(st[k], 1) for k in
                                  ("upload_ms", "prepare_ms", "search_ms", "remap_ms", "total_ms")}}
            return ptrh

        self.ptrh = build_index_bytes(n, dist, None, build=build, tag="str")
        self.idx = ph_gpu.PtrHashIndex(self.ptrh, device=dist.local)
        if cfg.get("layout") == "hot":
            self.idx.set_l2_policy(64 << 20, 0)  # hot-first + window
        self.nq = n
        self.data, self.offs = gen(1)  # the shuffled query stream
        self.bijective = True
        self.pin_data = torch.empty(self.data.numel(), dtype=torch.uint8).pin_memory()
        self.pin_data.copy_(self.data)
        self.pin_offs = torch.empty(n + 1, dtype=torch.int64).pin_memory()
        self.pin_offs.copy_(self.offs)
        nbytes = self.data.numel()
        self.stream_bytes = (nbytes + 8.0 * (n + 1)) / n + 4.0
        self.h2d, self.d2h = nbytes + 8 * (n + 1), n * 4
        self.api = "ph_gpu_index_stream_bytes (host pinned bytes + offsets -> host u32 out)"

    def query(self, out, minimal, stream):
        self.idx.query((self.data, self.offs), out=out, minimal=minimal, out_width=4,
                       stream=stream)

    def e2e(self, pin_out):
        self.idx.query((self.pin_data, self.pin_offs), out=pin_out, minimal=True, out_width=4)

    def reference_answers(self, ri, minimal, m):
        d = self.pin_data.numpy()
        o = self.pin_offs.numpy().view(np.uint64)[:m + 1]
        return ri.query_bytes(d, o, minimal, "single", threads=os.cpu_count() or 1)

    def cpu_runner(self, ri, S):
        """The reference's span<const std::string> bulk queries over std::strings made once
        from the first S queries of the stream (materialisation untimed)."""
        from oracle.bindings import RefStrings
        d = self.pin_data.numpy()
        o = np.ascontiguousarray(self.pin_offs.numpy().view(np.uint64)[:S + 1])
        sets = {}
        out = np.empty(S, dtype=np.uint64)

        def run(count, minimal, mode, width, threads):
            if count not in sets:
                sets[count] = RefStrings(ri.ref, d, o[:count + 1])
            sets[count].query(ri, minimal, mode, width, threads=threads, out=out[:count])

        def close():
            for v in sets.values():
                v.close()
        return run, ("queries of the same shuffled stream as std::string keys "
                     "(materialised before timing)"), close


class KmerWork:
    """config 5: k-mers of a packed DNA sequence, in sequence order, fused front end."""

    def __init__(self, args, cfg, dist, bench, sp):
        import torch
        from oracle.bindings import Ref
        from paper_2502_15539_b200 import ph_gpu
        self.cfg, self.k = cfg, cfg["k"]
        k = self.k
        self.n_bases = cfg["n"] + k - 1
        nw = (self.n_bases + 31) // 32
        self.seq = torch.empty(nw, dtype=torch.int64, device="cuda")
        assert bench.phb_gen_dna(C.c_void_p(self.seq.data_ptr()), C.c_uint64(nw),
                                 C.c_uint64(DNA_SEED + dist.rank), sp) == 0
        self.nq = self.n_bases - k + 1
        kmers = torch.empty(self.nq, dtype=torch.int64, device="cuda")
        assert bench.phb_kmers(C.c_void_p(self.seq.data_ptr()), C.c_uint64(self.n_bases), k,
                               C.c_void_p(kmers.data_ptr()), sp) == 0
        self.kmers_host = torch.empty(self.nq, dtype=torch.int64).pin_memory()
        self.kmers_host.copy_(kmers)

        def build():
            uniq = torch.unique(kmers)  # deduplicated key set, as the workload defines it
            self.n_unique = int(uniq.numel())
            hu = uniq.cpu().numpy().view(np.uint64)
            del uniq
            ref = Ref()
            log(f"[fixture] {self.nq} k-mers, {hu.size} distinct; reference build...")
            return ref.build_u64(hu, ref_params(ref), threads=0)

        self.n_unique = None
        self.ptrh = build_index_bytes(self.nq, dist, None, build=build, tag=f"kmer{k}")
        del kmers
        self.idx = ph_gpu.PtrHashIndex(self.ptrh, device=dist.local)
        if cfg.get("layout") == "file":
            self.idx.set_l2_policy(0, 2)  # file order: the partitioned path
        elif cfg.get("layout") == "hot":
            self.idx.set_l2_policy(64 << 20, 0)  # hot-first + window: the direct kernel
        self.n = int(self.idx.info.n)
        self.bijective = self.n == self.nq  # no duplicate k-mer: outputs are a permutation
        self.pin_seq = torch.empty(nw, dtype=torch.int64).pin_memory()
        self.pin_seq.copy_(self.seq)
        self.stream_bytes = 8.0 * nw / self.nq + 4.0  # 0.25 B packed bases + 4 B out
        self.h2d, self.d2h = nw * 8, self.nq * 4
        self.api = "ph_gpu_index_stream_kmers (host pinned packed sequence -> host u32 out)"

    def query(self, out, minimal, stream):
        self.idx.query_kmers(self.seq, self.n_bases, self.k, out=out, minimal=minimal,
                             out_width=4, stream=stream)

    def e2e(self, pin_out):
        self.idx.query_kmers(self.pin_seq, self.n_bases, self.k, out=pin_out, minimal=True,
                             out_width=4)

    def reference_answers(self, ri, minimal, m):
        kh = self.kmers_host.numpy().view(np.uint64)[:m]
        return ri.query_u64(kh, minimal, "stream", 32, threads=os.cpu_count() or 1)

    def cpu_runner(self, ri, S):
        sample = np.ascontiguousarray(self.kmers_host.numpy().view(np.uint64)[:S])
        out = np.empty(S, dtype=np.uint64)

        def run(count, minimal, mode, width, threads):
            ri.query_u64(sample[:count], minimal, mode, width, threads=threads, out=out[:count])
        return run, ("k-mers in sequence order, materialised as u64 keys (the reference has no "
                     "k-mer front end; extraction untimed)"), lambda: None


WORKLOADS = {"u64": U64Work, "str": StrWork, "kmer": KmerWork}


def run_ours(args, cfg):
    import torch
    dist = Dist("nccl")
    torch.cuda.set_device(dist.local)
    from paper_2502_15539_b200 import ph_gpu
    bench = C.CDLL(os.path.join(ROOT, "paper_2502_15539_b200", "libph_bench.so"))
    stream = torch.cuda.current_stream()
    sp = C.c_void_p(stream.cuda_stream)
    W = WORKLOADS[cfg["kind"]](args, cfg, dist, bench, sp)
    idx, info, nq, n = W.idx, W.idx.info, W.nq, int(W.idx.info.n)
    out = torch.empty(nq, dtype=torch.int32, device="cuda")
    out_nm = torch.empty(nq, dtype=torch.int32, device="cuda")

    # ---- correctness gate (untimed) ----
    W.query(out, True, stream.cuda_stream)
    W.query(out_nm, False, stream.cuda_stream)
    torch.cuda.synchronize()
    remap_frac = float((out_nm.to(torch.int64) & 0xFFFFFFFF).ge(n).double().mean().item())
    gate = {"remap_fraction": remap_frac}
    if W.bijective:
        bits = torch.zeros((n + 31) // 32, dtype=torch.int32, device="cuda")
        bad = torch.zeros(2, dtype=torch.int64, device="cuda")
        bench.phb_bijection(C.c_void_p(out.data_ptr()), C.c_uint64(nq), C.c_uint64(n),
                            C.c_void_p(bits.data_ptr()), C.c_void_p(bad.data_ptr()), sp)
        torch.cuda.synchronize()
        gate["bijection"] = bad.tolist() == [0, 0]
        del bits
    pin_o = torch.empty(nq, dtype=torch.int32).pin_memory()
    if args.verify != "none" and dist.rank == 0:
        from oracle.bindings import Ref
        ri = Ref().load(W.ptrh)
        m = nq if args.verify == "full" else min(nq, 10**7)
        t = time.time()
        ok = True
        for minimal, o in ((True, out), (False, out_nm)):
            want = W.reference_answers(ri, minimal, m)
            got = o[:m].cpu().numpy().view(np.uint32)
            ok &= bool(np.array_equal(got, want.astype(np.uint32))) and int(want.max()) < 2**32
            del want
        gate["bit_exact_vs_reference"] = ok
        gate["verified_queries"] = int(m) * 2
        log(f"[gate] {m} queries x (minimal, non-minimal) vs the reference: "
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

    def gather_rate(nbytes):  # G random 1-byte loads (sectors) / s over an nbytes buffer
        g_ms = time_ms(lambda: bench.phb_gather(C.c_void_p(pil.data_ptr()), C.c_uint64(nbytes),
                                                C.c_uint64(nl), C.c_uint64(1), 8, 8,
                                                C.c_void_p(sink.data_ptr()), sp))
        return nl / g_ms / 1e6

    r_gather = gather_rate(pil.numel())
    # the partitioned path's pass B gathers from one L2-resident slice (32 MiB) at a time
    slice_bytes = min(pil.numel(), 32 << 20)
    r_gather_slice = gather_rate(slice_bytes)
    # ... and shares the SM's L1->XBAR port with its own streams: the same gathers with 8 B
    # read and 4 B written per gather beside them (k_port, pass B's launch shape)
    r_port = None
    if cfg["kind"] != "str" and hasattr(bench, "phb_port_model"):
        bench.phb_port_model.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int,
                                         C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        p_in = torch.empty(nl, dtype=torch.int64, device="cuda")
        p_out = torch.empty(nl, dtype=torch.int32, device="cuda")
        run_port = lambda: bench.phb_port_model(  # noqa: E731
            C.c_void_p(pil.data_ptr()), C.c_uint64(slice_bytes), C.c_uint64(nl), C.c_uint64(1), 1, 42,
            C.c_void_p(p_in.data_ptr()), C.c_void_p(p_out.data_ptr()), C.c_void_p(sink.data_ptr()), sp)
        port_ms = time_ms(run_port, 3)
        r_port = nl / port_ms / 1e6
        del p_in, p_out
    del pil

    # ---- timed region: value ----
    sampler = ClockSampler(torch.cuda.current_device())
    sampler.start()

    def timed(minimal):
        for _ in range(args.warmup):
            W.query(out, minimal, stream.cuda_stream)
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
            W.query(out, minimal, stream.cuda_stream)
            b.record(stream)
            ms.append((a, b))
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        dist.barrier()
        sampler.window(t0, t1)
        return [a.elapsed_time(b) for a, b in ms], ph_gpu.launch_count() - l0

    ms_min, launches = timed(True)
    ms_nm, _ = timed(False)
    total_ms = dist.max(sum(ms_min))
    total_nm = dist.max(sum(ms_nm))

    # ---- per-pass times of the partitioned path (separate loop: events between passes) ----
    passes = None
    if cfg.get("layout") == "file" and info.pilot_bytes > (64 << 20):
        ph_gpu.set_pass_timing(True)
        for _ in range(args.steps):
            flush.zero_()
            W.query(out, True, stream.cuda_stream)
        torch.cuda.synchronize()
        sums, calls = ph_gpu.pass_times()
        ph_gpu.set_pass_timing(False)
        if calls:
            passes = [dist.max(x / calls) for x in sums]

    # ---- timed region: e2e through the public host API ----
    for _ in range(2):
        W.e2e(pin_o)
    dist.barrier()
    torch.cuda.synchronize()
    l0 = ph_gpu.launch_count()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        W.e2e(pin_o)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    e2e_launches = ph_gpu.launch_count() - l0
    dist.barrier()
    sampler.window(t0, t1)
    e2e_s = dist.max(t1 - t0)
    sampler.stop()
    W.query(out, True, stream.cuda_stream)  # e2e outputs must equal the device path's
    torch.cuda.synchronize()
    if not torch.equal(pin_o.cuda(), out):
        raise SystemExit("e2e host-path output differs from the device path")

    # ---- replay bound: the pilot gathers alone at the true bucket addresses ----
    replay = replay_bounds(W, idx, info, time_ms, cfg, args)

    # ---- report ----
    N, K = dist.world, args.steps
    value = N * nq * K / (total_ms * 1e-3) / 1e9
    step_ms = total_ms / K
    sectors = 1.0 + remap_frac * (1.0 + 32.0 / 44.0)  # pilot + CLEF (i>=12 touches 2nd sector)
    table_bytes = int(info.pilot_bytes) + int(info.remap_bytes)
    peak, peak_src = measured_peaks()
    in_bytes = W.stream_bytes - 4.0  # keys (8 B), packed bases (0.25 B) or string bytes+offsets
    partitioned = passes is not None
    if partitioned:
        # The path as built: pass A reads the input and writes (key, position)
        # entries (10 B), pass B reads the keys (8 B) and writes u32 slots (4 B), pass C reads
        # (slot, position) (6 B) and writes the output (4 B); the pilots and the remap table
        # come from DRAM once per step (their slices are L2-resident while pass B runs).
        per_key = {"A": in_bytes + 10.0, "B": 12.0, "C": 10.0}
        bytes_per_key = sum(per_key.values()) + table_bytes / nq
        dram_note = (f"path as built: pass A {per_key['A']:.2f} B (input + 10 B entry) + pass B "
                     f"12 B (8 B key + 4 B slot) + pass C 10 B (6 B entry + 4 B out) per query "
                     f"+ pilots and remap once per step ({table_bytes} B)")
    elif table_bytes <= (64 << 20):
        bytes_per_key = W.stream_bytes + table_bytes / nq
        dram_note = (f"{W.stream_bytes:.2f} B streamed per query + the L2-resident pilots and "
                     f"remap table once per step ({table_bytes} B); the binding bound is the L2 "
                     f"gather rate (dominant_kernel)")
    else:
        bytes_per_key = W.stream_bytes + 32.0 * sectors
        dram_note = (f"{W.stream_bytes:.2f} B streamed per query + 32 B x (1 pilot sector + "
                     f"remap_fraction x 1.727 CacheLineEF sectors) from DRAM")
    achieved = nq * bytes_per_key / (step_ms * 1e-3) / 1e9
    stream_ms = nq * W.stream_bytes / (bw_copy * 1e9) * 1e3
    gather_ms = nq * sectors / (r_gather * 1e9) * 1e3
    t_model = max(stream_ms, gather_ms)
    traffic, traffic_src = measured_traffic(args.config)
    cpu = None
    if dist.rank == 0 and N == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(W, args)
    dominant = None
    pass_block = None
    if partitioned:
        A, B, Cc = passes
        gathers_b = nq * sectors / (B * 1e-3) / 1e9
        pass_block = {
            "method": "CUDA events around the three passes on the query stream "
                      "(ph_gpu_set_pass_timing), mean over a separate loop of the same steps",
            "bin": {"kernel": "k_bin_tma", "ms": round(A, 4), "bound": "hbm",
                    "algorithmic_bytes_per_key": round(per_key["A"], 3),
                    "achieved_gbs": round(nq * per_key["A"] / A / 1e6, 1),
                    "frac": round(nq * per_key["A"] / A / 1e6 / peak, 4)},
            "query": {"kernel": "k_query_regions", "ms": round(B, 4),
                      "bound": "L1->XBAR request port: one L2 request per pilot gather from "
                               "the L2-resident slice, sharing the port with the pass's own "
                               "8 B in + 4 B out per key",
                      "gathers_gsectors_s": round(gathers_b, 2),
                      "peak_gsectors_s": round(r_port or r_gather_slice, 2),
                      "peak_source": (f"live k_port microbenchmark: random 1-byte gathers over "
                                      f"{slice_bytes >> 20} MiB with 8 B streamed in and 4 B out "
                                      f"per gather, two outputs per store like the pass "
                                      f"(tools/port_model.py, DESIGN.md §3)"
                                      if r_port else
                                      f"live k_gather microbenchmark over {slice_bytes >> 20} MiB"),
                      "frac": round(gathers_b / (r_port or r_gather_slice), 4),
                      "gather_only_peak_gsectors_s": round(r_gather_slice, 2),
                      "frac_vs_gather_only": round(gathers_b / r_gather_slice, 4),
                      "hbm_bytes_per_key": 12.0,
                      "hbm_frac": round(nq * 12.0 / B / 1e6 / peak, 4)},
            "unbin": {"kernel": "k_unbin_tma", "ms": round(Cc, 4), "bound": "hbm",
                      "algorithmic_bytes_per_key": 10.0,
                      "achieved_gbs": round(nq * 10.0 / Cc / 1e6, 1),
                      "frac": round(nq * 10.0 / Cc / 1e6 / peak, 4)},
        }
        k = max(("bin", "query", "unbin"), key=lambda x: pass_block[x]["ms"])
        pass_block["dominant"] = k
        dominant = dict(pass_block[k], share_of_step=round(pass_block[k]["ms"] / step_ms, 4))
    elif table_bytes <= (64 << 20) and cfg["kind"] != "str":
        g_s = nq * sectors / step_ms / 1e6
        dominant = {"kernel": "k_query_u64", "ms": round(step_ms, 4),
                    "bound": "L1->XBAR request port: one L2 request per pilot gather (pilots "
                             "L2-resident), sharing the port with the 8 B in + 4 B out per key",
                    "gathers_gsectors_s": round(g_s, 2),
                    "peak_gsectors_s": round(r_port or r_gather, 2),
                    "peak_source": (f"live k_port microbenchmark: random 1-byte gathers over "
                                    f"{slice_bytes} B with 8 B streamed in and 4 B out per gather"
                                    if r_port else
                                    f"live k_gather microbenchmark over {int(info.pilot_bytes)} B"),
                    "frac": round(g_s / (r_port or r_gather), 4),
                    "gather_only_peak_gsectors_s": round(r_gather, 2),
                    "frac_vs_gather_only": round(g_s / r_gather, 4)}
    elif cfg["kind"] == "str":
        # The string kernel is bound by the SM's L1 data pipe: one wavefront per
        # cycle per SM. Wavefronts per key come from the committed ncu capture of this kernel on
        # this fixture (profiles/r02_traffic.json); the time and the clock are this run's.
        wf = lsu_wavefronts("config4", "k_query_bytes")
        clk = sampler.summary().get("sm_mhz")
        if wf and clk:
            sms_n = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
            per_key = wf * sms_n / cfg["n"]
            rate = nq * per_key / (step_ms * 1e-3) / (sms_n * clk * 1e6)
            dominant = {"kernel": "k_query_bytes", "ms": round(step_ms, 4),
                        "bound": "L1 data pipe: shared-memory T-table reads (16 per AES round) and the "
                                 "per-lane key-byte loads, one wavefront per cycle per SM",
                        "wavefronts_per_key": round(per_key, 3),
                        "wavefronts_source": "ncu l1tex__data_pipe_lsu_wavefronts of this kernel on this "
                                             "fixture (profiles/r02_ncu_full_query_config4_raw.csv)",
                        "achieved_wavefronts_per_clk_per_sm": round(rate, 4), "peak": 1.0,
                        "sm_mhz": clk, "frac": round(rate, 4)}
    res = {
        "metric": METRIC,
        "value": round(value, 3),
        "unit": "Gkeys/s",
        "ns_per_key": round(1.0 / value, 5),
        "n_gpus": N,
        "steps": K,
        "warmup": args.warmup,
        "ms_per_step": round(step_ms, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u64",
        "data": "synthetic (seeded generators, SURVEY §8d; index built by the reference builder)",
        "config": config_dict(cfg, W.ptrh, N),
        "setup": {"pilot_layout": ("file order, partitioned path" if partitioned
                                   else "hot-first + persisting window" if cfg.get("layout") == "hot"
                                   else "library default (file order)"),
                  "l2": "flushed between steps (512 MiB write, outside the timed events)"},
        "nonminimal": {"value": round(N * nq * K / (total_nm * 1e-3) / 1e9, 3), "unit": "Gkeys/s",
                       "ms_per_step": round(total_nm / K, 4)},
        "gpu_launches": int(launches),
        "e2e": {"value": round(N * nq * K / e2e_s / 1e9, 4), "unit": "Gkeys/s",
                "h2d_bytes_per_step": int(W.h2d), "d2h_bytes_per_step": int(W.d2h),
                "api": W.api, "gpu_launches": int(e2e_launches)},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                     "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": traffic,
                     "traffic_source": traffic_src,
                     "scope": ("the whole query step (passes A+B+C)" if partitioned
                               else "the query kernel"),
                     "peak_source": peak_src,
                     "algorithmic_bytes_per_key": round(bytes_per_key, 3),
                     "note": dram_note,
                     "frac_vs_stream_floor": round(stream_ms / step_ms, 4),
                     "stream_floor": f"{W.stream_bytes:.2f} B/query (input + u32 out) at the "
                                     f"live copy bandwidth {bw_copy:.0f} GB/s: "
                                     f"{stream_ms:.4f} ms"},
        "dominant_kernel": dominant,
        "uniform_gather_model": {
            "what": "SURVEY §8d / BASELINE.md §2: max(stream bytes / copy bandwidth, pilot + "
                    "remap sectors / uniform random-gather rate over the whole pilot array); "
                    "the skewed cubic-gamma access and the partitioned path both beat it",
            "t_model_ms": round(t_model, 4), "t_measured_ms": round(step_ms, 4),
            "speedup_vs_model": round(t_model / step_ms, 4),
            "additive_bound_ms": round(stream_ms + gather_ms, 4),
            "stream_bound_ms": round(stream_ms, 4), "gather_bound_ms": round(gather_ms, 4),
            "copy_gbs": round(bw_copy, 1), "r_gather_gsectors_s": round(r_gather, 3),
            "gather_buffer_bytes": int(info.pilot_bytes)},
        "replay": replay,
        "partition_passes": pass_block,
        "construction": getattr(W, "construction", None),
        "gate": gate,
        "clocks": sampler.summary(),
        "cpu_baseline": cpu,
    }
    # free this config's device and pinned memory before the secondary configs run
    del W, idx, out, out_nm, pin_o, flush
    ph_gpu_trim_all()
    if dist.rank == 0 and N == 1 and args.secondary_configs and args.config == 3:
        res["secondary"] = run_secondaries(args)
    if dist.rank == 0:
        print(json.dumps(res), flush=True)
    dist.close()


def ph_gpu_trim_all():
    import gc

    import torch
    gc.collect()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()


def lsu_wavefronts(config_key: str, kernel: str):
    """L1 data-pipe wavefronts per SM of `kernel` from the committed ncu capture, or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_traffic.json")) as f:
            return json.load(f)[config_key]["kernels"][kernel].get("lsu_wavefronts_per_sm")
    except (OSError, KeyError, ValueError):
        return None


def measured_traffic(config: int):
    """DRAM bytes per step (dram__bytes_read.sum + dram__bytes_write.sum over the step's
    kernels) from the committed ncu capture of this bench's own command on its own fixture
    (profiles/r02_traffic.json, written by tools/traffic_from_ncu.py)."""
    prof = os.path.join(ROOT, "profiles", "r02_traffic.json")
    try:
        with open(prof) as f:
            d = json.load(f).get(f"config{config}")
        return int(d["dram_bytes_per_step"]), d["source"]
    except Exception:
        return None, None


def replay_bounds(W, idx, info, time_ms, cfg, args):
    """The pilot reads alone (ph_gpu_gather_replay_u64) at the index's true bucket addresses:
    in query order (the direct kernel's access pattern) and, for the partitioned path, with
    the keys stably sorted by partition group (pass B's access pattern). u64 / k-mer configs."""
    import torch
    keys = getattr(W, "q", None)
    if cfg["kind"] == "kmer":
        keys = torch.from_numpy(W.kmers_host.numpy()).cuda()
    if keys is None or args.no_replay:
        return None
    nq = keys.numel()
    res = {"what": "ph_gpu_gather_replay_u64: key stream (8 B) + one pilot gather per key at "
                   "the true bucket address, no slot arithmetic / remap / output",
           "direct_order_ms": round(time_ms(lambda: idx.gather_replay(keys)), 4)}
    pb = int(info.pilot_bytes)
    if pb > (64 << 20):
        G = max(2, -(-pb // (32 << 20)))  # ph_abi.cu partition_groups (32 MiB slices)
        C_ = 0x517CC1B727220A95  # kMixConstant (hash.hpp:13), < 2^63
        seed = int(info.seed)
        seed = seed - (1 << 64) if seed >= (1 << 63) else seed
        h = (keys ^ seed) * C_  # wrapping int64 multiply = hash_int (hash.hpp:27)
        g = (((h >> 32) & 0xFFFFFFFF) * G) >> 32
        del h
        order = torch.sort(g, stable=True).indices
        del g
        grouped = keys[order]
        del order
        res["grouped_order_ms"] = round(time_ms(lambda: idx.gather_replay(grouped)), 4)
        res["groups"] = G
        del grouped
    res["gathers_per_step"] = nq
    return res


def run_secondaries(args):
    """Configs 4 (strings) and 5 (k-mers) in their own processes (same steps / warm-up, full
    gate, CPU matrix), so the driver's default run carries their numbers next to config 3."""
    import subprocess
    out = {}
    for c in (4, 5):
        if c == args.config:
            continue
        cmd = [sys.executable, os.path.abspath(__file__), "--config", str(c), "--steps",
               str(args.steps), "--warmup", str(args.warmup), "--verify", args.verify,
               "--cpu-sample", str(args.cpu_sample), "--no-secondary"]
        t = time.time()
        p = subprocess.run(cmd, capture_output=True, text=True)
        sys.stderr.write(p.stderr[-4000:])
        lines = [x for x in p.stdout.splitlines() if x.startswith("{")]
        if p.returncode == 0 and lines:
            d = json.loads(lines[-1])
            d["driver_note"] = f"run by bench.py as a subprocess in {time.time() - t:.0f} s"
            out[f"config{c}"] = d
        else:
            out[f"config{c}"] = {"error": f"rc={p.returncode}", "stderr": p.stderr[-1500:]}
    return out


CPU_MODES = (("loop", 0), ("stream", 32), ("batched", 64))  # ptrhash.cpp:160-174 run_mode


def time_best(fn, reps=3):
    """One warm-up, then the best of `reps` (proj/tools/ptrhash.cpp:212-223)."""
    fn()
    best = 1e30
    for _ in range(reps):
        t = time.perf_counter()
        fn()
        best = min(best, time.perf_counter() - t)
    return best


def cpu_baseline(W, args):
    """The reference's own CPU query path on this box's host cores (SURVEY
    §8d): T = 1 and T = all hardware threads x index_loop / index_stream(32) /
    index_batched(64) x minimal / non-minimal, contiguous slices per thread as the CLI bench
    does (ptrhash.cpp:486-512), one warm-up and the best of 3 (:212-223), each cell on a
    bounded sample of this config's query stream. `value` is the T = all, index_stream(32),
    minimal cell (the reference's recommended bulk query)."""
    from oracle.bindings import Ref
    ri = Ref().load(W.ptrh)
    T = os.cpu_count() or 1
    S_all = min(W.nq, args.cpu_sample if W.cfg["kind"] != "str" else args.cpu_sample // 4)
    S_one = min(S_all, max(args.cpu_sample // 50, 1))
    run, what, close = W.cpu_runner(ri, S_all)
    cells = []
    t0 = time.time()
    for threads, S in ((1, S_one), (T, S_all)):
        for mode, width in CPU_MODES:
            for minimal in (True, False):
                sec = time_best(lambda: run(S, minimal, mode, width, threads))
                cells.append({"threads": threads, "mode": mode if not width else f"{mode}:{width}",
                              "minimal": minimal, "ns_per_key": round(sec / S * 1e9, 3),
                              "gkeys_s": round(S / sec / 1e9, 4), "sample": S})
    close()
    ri.close()
    head = next(c for c in cells if c["threads"] == T and c["mode"] == "stream:32" and c["minimal"])
    log(f"[cpu] reference matrix ({len(cells)} cells) in {time.time() - t0:.1f}s")
    return {"value": head["gkeys_s"], "unit": "Gkeys/s", "ns_per_key": head["ns_per_key"],
            "cores": T, "kind": "reference", "cpu_model": cpu_model(),
            "sample": (f"first {S_all} {what}; reference PtrHashIndex::index_stream(lookahead "
                       f"32), minimal, {T} threads, contiguous slices, best of 3 after 1 "
                       f"warm-up (the full matrix is in `matrix`; T=1 cells use the first "
                       f"{S_one})"),
            "matrix": cells}


# ---------------------------------------------------------------------------
# reference arm
# ---------------------------------------------------------------------------
def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle.bindings import Port, Ref
    ref, port = Ref(), Port()
    T = os.cpu_count() or 1
    t = time.time()
    S = min(cfg["n"], args.cpu_sample)
    kind = cfg["kind"]
    if kind == "u64":
        n = cfg["n"]
        keys = port.gen_keys("corpus", 0, n, n, GEN_SEED)
        ptrh = ref.build_u64(keys, ref_params(ref), threads=0)
        del keys
        perm = cfg["order"] == "perm"
        q = port.gen_keys("perm" if perm else "sample", 0, S, n, GEN_SEED,
                          PERM_SEED if perm else SAMPLE_SEED)
        ri = ref.load(ptrh)
        out = np.empty(S, dtype=np.uint64)
        step = lambda: ri.query_u64(q, True, "stream", 32, threads=T, out=out)  # noqa: E731
        what = "index_stream(lookahead 32)"
    elif kind == "str":
        n = cfg["n"]
        data, offs = port.gen_strings(0, n, n, STR_SEED)
        ptrh = ref.build_bytes(data, offs, ref_params(ref), lean=True)
        del data, offs
        from oracle.bindings import RefStrings
        S = min(n, args.cpu_sample // 4)  # as our arm's cpu_baseline (std::string keys)
        qd, qo = port.gen_strings(0, S, n, STR_SEED, PERM_SEED)
        ri = ref.load(ptrh)
        out = np.empty(S, dtype=np.uint64)
        rs = RefStrings(ref, qd, qo)  # std::string keys made before timing
        step = lambda: rs.query(ri, True, "stream", 32, threads=T, out=out)  # noqa: E731
        what = "index_stream(lookahead 32) over std::string keys"
    else:
        k = cfg["k"]
        n_bases = cfg["n"] + k - 1
        seq = port.gen_dna(n_bases, DNA_SEED)
        kmers = port.kmers(seq, n_bases, k)
        try:
            ptrh = ref.build_u64(kmers, ref_params(ref), threads=0)
        except RuntimeError:  # duplicate k-mers: build over the distinct ones
            ptrh = ref.build_u64(np.unique(kmers), ref_params(ref), threads=0)
        q = np.ascontiguousarray(kmers[:S])
        del kmers
        ri = ref.load(ptrh)
        out = np.empty(S, dtype=np.uint64)
        step = lambda: ri.query_u64(q, True, "stream", 32, threads=T, out=out)  # noqa: E731
        what = "index_stream(lookahead 32) over materialised k-mers"
    log(f"[reference] fixture + index built in {time.time() - t:.1f}s")
    for _ in range(args.warmup):
        step()
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        step()
        ts.append(time.perf_counter() - t0)
    total = sum(ts)
    value = S * args.steps / total / 1e9
    sample = (f"first {S} queries of the config's query stream per step; reference "
              f"PtrHashIndex::{what}, minimal, {T} threads, contiguous slices")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(value, 5), "unit": "Gkeys/s",
        "ns_per_key": round(1 / value, 4), "n_gpus": int(os.environ.get("WORLD_SIZE", "1")),
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(total / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": config_dict(cfg, ptrh, int(os.environ.get("WORLD_SIZE", "1"))),
        "reference_sample": (f"each step times the first {S} of the {cfg['nq']} queries of the "
                             f"same stream; Gkeys/s is per query, so it compares with our "
                             f"arm's whole-stream steps"),
        "cpu_baseline": {"value": round(value, 5), "unit": "Gkeys/s", "cores": T,
                         "kind": "reference", "cpu_model": cpu_model(), "sample": sample},
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
    ap.add_argument("--no-replay", action="store_true")
    ap.add_argument("--no-construction", dest="construction", action="store_false",
                    help="skip the construction comparison (ph_gpu_build_u64 vs the reference)")
    ap.add_argument("--no-secondary", dest="secondary_configs", action="store_false",
                    help="do not run configs 4 and 5 after the main config (N=1)")
    ap.add_argument("--layout", default="", choices=["", "file", "hot", "default"],
                    help="override the config's pilot layout (file: partitioned path when large; "
                         "hot: hot-first layout + persisting window, the direct kernel)")
    args = ap.parse_args()
    if args.warmup < 3:
        log("note: warmup raised to 3 (timing rules)")
        args.warmup = 3
    cfg = dict(CONFIGS[args.config])
    cfg["nq"] = cfg["n"]  # queries per step: every config queries n keys (k-mers: n windows)
    if args.layout:
        cfg["layout"] = args.layout
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
