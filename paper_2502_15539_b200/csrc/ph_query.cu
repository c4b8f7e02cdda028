// ph_query.cu — the bulk query kernels (sm_100a).
//
// One kernel answers a batch of keys exactly as PtrHashIndex::index_loop /
// index_stream / index_batched do (/root/reference/proj/src/index.cpp:15-137):
//   out[i] = minimal ? remap_slot(slot_of(hash(keys[i]))) : slot_of(hash(keys[i]))
//
// Work decomposition: a warp owns a tile of 32*KPT consecutive
// keys; lane l handles keys tile + j*32 + l for j < KPT, so every key load and
// every output store is one coalesced 256-B / 128-B warp access. Per thread,
// all KPT pilot addresses are computed first and the KPT independent 1-byte
// gathers are issued back to back before any is consumed: this is the GPU's
// version of the CPU's prefetch ring (index.cpp:101-135), with
// KPT * (resident warps) gathers in flight per SM. The rare slot >= n keys
// (~1%) are compacted across the warp with __ballot_sync so one convergent
// round of remap decodes serves the whole tile.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

#include "ph_device.cuh"
#include "ph_kernels.h"

namespace phg {

// Compile-time switches for tools/tune.py variant builds (keys per thread and CTAs per SM
// are per-regime template parameters, see launch_u64_t).
#ifndef PH_PIPE
#define PH_PIPE 1
#endif
// deferred remap (warp-private lists + k_remap_patch) compiled in
#ifndef PH_DEFER
#define PH_DEFER 1
#endif
#ifndef PH_THREADS
#define PH_THREADS 128
#endif
// L2-resident tuning: keys per thread and CTAs per SM
#ifndef PH_L2_KPT
#define PH_L2_KPT 4
#endif
#ifndef PH_L2_MINB
#define PH_L2_MINB 8
#endif

// k-mer key of window i of a 2-bit packed sequence (word w holds bases 32w..32w+31,
// base 32w+t at bits 2(31-t), i.e. MSB-first): the k bases starting at i packed with the
// first base in the most significant bits (A=0, C=1, G=2, T=3), as the k-mer workload of
// BASELINE.json defines its u64 keys. nwords bounds the second word read.
__device__ __forceinline__ uint64_t kmer_at(const uint64_t* __restrict__ seq, uint64_t nwords,
                                            uint64_t i, uint32_t kbits) {
    const uint64_t a = i >> 5;
    const uint32_t o = (uint32_t)(i & 31) * 2;
    const uint64_t wa = __ldg(seq + a);
    const uint64_t wb = (o && a + 1 < nwords) ? __ldg(seq + a + 1) : 0;
    const uint64_t top = o ? (wa << o) | (wb >> (64 - o)) : wa;
    return kbits == 64 ? top : top >> (64 - kbits);
}

// SRC = 0: keys[] is an array of u64 keys. SRC = 1: keys[] is a 2-bit packed sequence of
// seq_words words and key i is its i-th k-mer (kbits = 2k) — the fused streaming front
// end for k-mer workloads: 0.25 B/query of input instead of 8 B.
// Deferred remap: the keys with slot >= n are appended to the warp's private list and
// decoded by k_remap_patch after the main kernel, so the dependent remap read leaves the
// main kernel's critical path (no third serial memory latency per tile). Ranks come from
// the same ballots as the inline path; the warp's running count stays in a register (no
// atomics). Entries beyond the list's capacity are decoded inline, never dropped.
template <int KPT, class OutT>
__device__ __forceinline__ void defer_tile(const DevIndex& ix, uint64_t* __restrict__ lidx,
                                           uint64_t* __restrict__ lrem, uint32_t lcap,
                                           uint32_t& wcount, const bool (&need)[KPT],
                                           uint64_t (&slot)[KPT], uint64_t base) {
    const unsigned lane = threadIdx.x & 31;
    const unsigned lt_mask = (1u << lane) - 1;
    unsigned m[KPT];
    uint32_t total = 0;
#pragma unroll
    for (int j = 0; j < KPT; j++) {
        m[j] = __ballot_sync(kFull, need[j]);
        total += __popc(m[j]);
    }
    if (total == 0) return;                 // warp-uniform
    if (wcount + total > lcap) {            // list full: decode this tile inline
        remap_tile<KPT, OutT>(ix, need, slot);
        return;
    }
    uint32_t pos = wcount;
#pragma unroll
    for (int j = 0; j < KPT; j++) {
        if (need[j]) {
            const uint32_t p = pos + __popc(m[j] & lt_mask);
            lidx[p] = base + (uint64_t)j * 32 + lane;
            lrem[p] = slot[j] - ix.n;
        }
        pos += __popc(m[j]);
    }
    wcount = pos;
}

// One warp per list: decode its entries and patch the outputs.
template <class OutT>
__global__ void __launch_bounds__(256) k_remap_patch(const DevIndex ix, const RemapList rl,
                                                     uint32_t nlists, OutT* __restrict__ out) {
    const uint32_t lcap = (uint32_t)(rl.cap / nlists);
    const unsigned lane = threadIdx.x & 31;
    for (uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < nlists;
         w += (gridDim.x * blockDim.x) >> 5) {
        const uint32_t c = min(rl.counts[w], lcap);
        const uint64_t* li = rl.idx + (uint64_t)w * lcap;
        const uint64_t* lr = rl.rem + (uint64_t)w * lcap;
        // four entries per lane in flight: the list reads, the decodes' table reads and the
        // patch stores of a round are independent (a list holds ~200 entries at config 2)
        for (uint32_t e0 = 0; e0 < c; e0 += 128) {
            uint64_t i4[4], r4[4];
#pragma unroll
            for (int q = 0; q < 4; q++) {
                const uint32_t e = e0 + q * 32 + lane;
                i4[q] = e < c ? li[e] : 0;
                r4[q] = e < c ? lr[e] : 0;
            }
#pragma unroll
            for (int q = 0; q < 4; q++) {
                const uint32_t e = e0 + q * 32 + lane;
                if (e < c) out[i4[q]] = (OutT)remap_get(ix, r4[q]);  // remap_slot, index.hpp:98-100
            }
        }
    }
}

// HOTF: the device pilots use the hot-first layout (pilot_offset); otherwise the file's
// own order, offset = part * B + bucket.
template <int G, bool POW2, class OutT, int KPT, int SRC, int MINB, bool DEFER, bool HOTF>
__global__ void __launch_bounds__(PH_THREADS, MINB) k_query_u64(const DevIndex ix,
                                                   const uint64_t* __restrict__ keys,
                                                   OutT* __restrict__ out, uint64_t nkeys_arg,
                                                   int minimal, uint64_t seq_words,
                                                   uint32_t kbits, const RemapList rl) {
    constexpr uint64_t kTile = 32ull * KPT;
    const uint64_t nkeys = nkeys_arg;
    const unsigned lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t pol_stream = policy_evict_first();
    // pass B of the partitioned path processes one L2-sized pilot slice after another:
    // evict_last would leave earlier slices' lines pinned, so it uses evict_normal
    const uint64_t pol_keep = ix.pilot_evict_normal ? policy_evict_normal() : policy_evict_last();

    const uint64_t stride = nwarps * kTile;
    const uint32_t P32 = (uint32_t)ix.P, B32 = (uint32_t)ix.B, S32 = (uint32_t)ix.S;
    // deferred-remap list of this warp (when rl.idx != nullptr)
    const uint32_t lcap = rl.idx ? (uint32_t)(rl.cap / nwarps) : 0;
    uint64_t* lidx = rl.idx ? rl.idx + warp * lcap : nullptr;
    uint64_t* lrem = rl.idx ? rl.rem + warp * lcap : nullptr;
    uint32_t wcount = 0;
    // PH_PIPE: the next tile's keys are loaded before this tile's pilot gather and remap,
    // so the key stream's DRAM latency overlaps them (software pipelining across tiles).
    uint64_t knext[KPT];
    // In-tile bounds as one 32-bit compare per element: rem = keys left in this tile.
    auto tile_rem = [&](uint64_t b) -> uint32_t {
        return b + kTile <= nkeys ? (uint32_t)kTile : (uint32_t)(nkeys - b);
    };
    auto load_keys = [&](uint64_t b, uint64_t (&k)[KPT]) {
        const uint32_t rem = tile_rem(b);
        if constexpr (SRC == 1) {
#pragma unroll
            for (int j = 0; j < KPT; j++)
                k[j] = (uint32_t)(j * 32) + lane < rem
                           ? kmer_at(keys, seq_words, b + (uint64_t)j * 32 + lane, kbits)
                           : 0;
        } else {
            const uint64_t* kp = keys + b + lane;
#pragma unroll
            for (int j = 0; j < KPT; j++)
                k[j] = (uint32_t)(j * 32) + lane < rem ? ld_stream_u64(kp + j * 32, pol_stream) : 0;
        }
    };
    if (PH_PIPE) load_keys(warp * kTile, knext);

    for (uint64_t base = warp * kTile; base < nkeys; base += stride) {
        const uint32_t rem = tile_rem(base);
        uint64_t h[KPT];
        if (PH_PIPE) {
#pragma unroll
            for (int j = 0; j < KPT; j++) h[j] = knext[j];
            if (base + stride < nkeys) load_keys(base + stride, knext);
        } else {
            load_keys(base, h);
        }
#pragma unroll
        for (int j = 0; j < KPT; j++) h[j] = kC * (h[j] ^ ix.seed);  // hash_int, hash.hpp:27
        uint32_t part[KPT];
        uint32_t pilot[KPT];
#pragma unroll
        for (int j = 0; j < KPT; j++) {
            // part_and_bucket, bucket_fn.hpp:66-72 (P, B < 2^32: checked at create)
            uint64_t x;
            part[j] = (uint32_t)mul32x64(P32, h[j], x);
            const uint32_t bucket = bucket_of<G>(x, B32, ix.opt_table);
            if (HOTF) {
                const bool hot = bucket < ix.hot_b;
                pilot[j] = ld_gather_u8(ix.pilots + pilot_offset(ix, part[j], bucket),
                                        (hot || !ix.cold_evict_first) ? pol_keep : pol_stream);
            } else {
                pilot[j] = ld_gather_u8(ix.pilots + ((uint64_t)part[j] * B32 + bucket), pol_keep);
            }
        }
        uint64_t slot[KPT];
        bool need[KPT];
#pragma unroll
        for (int j = 0; j < KPT; j++) {
            // slot_of, index.hpp:91-96
            slot[j] = (uint64_t)part[j] * S32 + reduce<POW2>(ix, h[j] ^ hash_pilot(ix, pilot[j]));
            need[j] = minimal && slot[j] >= ix.n && (uint32_t)(j * 32) + lane < rem;
        }
        if (minimal) {  // remap_slot, index.hpp:98-100
            if (DEFER && rl.idx) defer_tile<KPT, OutT>(ix, lidx, lrem, lcap, wcount, need, slot, base);
            else remap_tile<KPT, OutT>(ix, need, slot);
        }
        OutT* op = out + base + lane;
#pragma unroll
        for (int j = 0; j < KPT; j++)
            if ((uint32_t)(j * 32) + lane < rem) st_stream(op + j * 32, slot[j]);
    }
    if (DEFER && rl.idx && lane == 0) rl.counts[warp] = wcount;
}

// ---------------------------------------------------------------------------
// launch plumbing
// ---------------------------------------------------------------------------
static std::atomic<uint64_t> g_launches{0};
static int g_threads_override = 0;
static int g_bps_override = 0;

uint64_t launch_count() { return g_launches.load(); }
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
void set_launch(int threads, int bps) {
    g_threads_override = threads;
    g_bps_override = bps;
}

template <class K>
static int grid_for(K kernel, int threads, uint64_t work_items_per_block, uint64_t nitems,
                    int device_sms) {
    int bps = g_bps_override;
    if (bps <= 0) {
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kernel, threads, 0) != cudaSuccess ||
            bps <= 0)
            bps = 1;
    }
    const uint64_t want = (nitems + work_items_per_block - 1) / work_items_per_block;
    const uint64_t cap = (uint64_t)device_sms * (uint64_t)bps;
    return (int)(want < cap ? (want ? want : 1) : cap);
}

// Key-source arguments of one launch: an array of u64 keys, or the k-mers of a packed
// 2-bit sequence (seq_words words, kbits = 2k).
struct KeySrc {
    const uint64_t* ptr;
    int kind;  // 0 = u64 array, 1 = k-mers
    uint64_t seq_words;
    uint32_t kbits;
};

// Two tunings of the same kernel, chosen per index by the pilot array's size
// (tools/tune.py sweeps); the L2 tuning assumes the file-order pilot layout
// (a hot-first layout only exists for DRAM-sized pilot arrays):
//  * DRAM regime (pilots > kDramRegimeBytes, e.g. configs 3/5): the pilot gather is bound
//    by DRAM row activations; KPT=8 with the compiler's register allocation (12 warps/SM)
//    and the inline warp-compacted remap measured fastest;
//  * L2 regime (pilots L2-resident, configs 1/2): latency-bound; KPT=4 at 8 CTAs/SM
//    (32 warps/SM) with the remap deferred to k_remap_patch measured fastest.
constexpr uint64_t kDramRegimeBytes = uint64_t{64} << 20;
static int g_regime = 0;  // 0 auto, 1 force L2 regime (file-order layouts), 2 force DRAM regime
void set_regime(int r) { g_regime = r; }

template <int G, bool POW2, class OutT, int SRC, int KPT, int MINB, bool DEFER, bool HOTF>
static cudaError_t launch_u64_k(const DevIndex& ix, const KeySrc& src, void* out, uint64_t n,
                                int minimal, cudaStream_t s, int sms, const RemapList& rl) {
    auto kern = k_query_u64<G, POW2, OutT, KPT, SRC, MINB, (PH_DEFER && DEFER), HOTF>;
    const int threads = g_threads_override > 0 ? g_threads_override : PH_THREADS;
    const int blocks = grid_for(kern, threads, (uint64_t)threads / 32 * 32 * KPT, n, sms);
    const uint32_t nlists = (uint32_t)blocks * (uint32_t)(threads / 32);
    const RemapList use = (PH_DEFER && DEFER && minimal && rl.idx && nlists <= kMaxRemapLists &&
                           rl.cap / nlists >= 32)
                              ? rl
                              : RemapList{nullptr, nullptr, nullptr, 0};
    cudaError_t e = launch_ex(ix, kern, blocks, threads, s, ix, src.ptr, static_cast<OutT*>(out), n,
                              minimal, src.seq_words, src.kbits, use);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    if (e == cudaSuccess && use.idx) {
        k_remap_patch<OutT><<<(nlists + 7) / 8, 256, 0, s>>>(ix, use, nlists,
                                                              static_cast<OutT*>(out));
        g_launches.fetch_add(1, std::memory_order_relaxed);
        e = cudaGetLastError();
    }
    return e;
}

template <int G, bool POW2, class OutT, int SRC>
static cudaError_t launch_u64_t(const DevIndex& ix, const KeySrc& src, void* out, uint64_t n,
                                int minimal, cudaStream_t s, int sms, const RemapList& rl) {
    const bool hotf = ix.hot_b < ix.B;
    {
        const bool dram = hotf || g_regime == 2 ||
                          (g_regime == 0 && ix.P * ix.B > kDramRegimeBytes);
        if (dram && hotf)
            return launch_u64_k<G, POW2, OutT, SRC, 8, 1, false, true>(ix, src, out, n, minimal, s,
                                                                       sms, rl);
        if (dram)
            return launch_u64_k<G, POW2, OutT, SRC, 8, 1, false, false>(ix, src, out, n, minimal,
                                                                        s, sms, rl);
        return launch_u64_k<G, POW2, OutT, SRC, PH_L2_KPT, PH_L2_MINB, true, false>(ix, src, out, n, minimal, s,
                                                                   sms, rl);
    }
}

template <class OutT, int SRC>
static cudaError_t launch_u64_w(const DevIndex& ix, int gamma_kind, bool pow2, const KeySrc& k,
                                void* o, uint64_t n, int minimal, cudaStream_t s, int sms,
                                const RemapList& rl) {
#define PH_CASE(G)                                                                          \
    case G:                                                                                 \
        return pow2 ? launch_u64_t<G, true, OutT, SRC>(ix, k, o, n, minimal, s, sms, rl)  \
                    : launch_u64_t<G, false, OutT, SRC>(ix, k, o, n, minimal, s, sms, rl);
    switch (gamma_kind) {
        PH_CASE(0)
        PH_CASE(1)
        PH_CASE(2)
        PH_CASE(3)
        PH_CASE(4)
    }
#undef PH_CASE
    return cudaErrorInvalidValue;
}

static cudaError_t launch_src(const DevIndex& ix, int gamma_kind, bool pow2, const KeySrc& k,
                              void* out, int out_width, uint64_t n, int minimal, cudaStream_t s,
                              int sms, const RemapList& rl) {
    if (n == 0) return cudaSuccess;
    if (k.kind == 1)
        return out_width == 4
                   ? launch_u64_w<uint32_t, 1>(ix, gamma_kind, pow2, k, out, n, minimal, s, sms, rl)
                   : launch_u64_w<uint64_t, 1>(ix, gamma_kind, pow2, k, out, n, minimal, s, sms, rl);
    return out_width == 4
               ? launch_u64_w<uint32_t, 0>(ix, gamma_kind, pow2, k, out, n, minimal, s, sms, rl)
               : launch_u64_w<uint64_t, 0>(ix, gamma_kind, pow2, k, out, n, minimal, s, sms, rl);
}

cudaError_t launch_query_u64(const DevIndex& ix, int gamma_kind, bool pow2, const uint64_t* keys,
                             void* out, int out_width, uint64_t n, int minimal, cudaStream_t s,
                             int sms, const RemapList& rl) {
    return launch_src(ix, gamma_kind, pow2, KeySrc{keys, 0, 0, 0}, out, out_width, n, minimal, s,
                      sms, rl);
}

cudaError_t launch_query_kmers(const DevIndex& ix, int gamma_kind, bool pow2, const uint64_t* seq,
                               uint64_t n_bases, int k, void* out, int out_width, int minimal,
                               cudaStream_t s, int sms, const RemapList& rl) {
    if (n_bases < (uint64_t)k) return cudaSuccess;
    const uint64_t n = n_bases - (uint64_t)k + 1;
    return launch_src(ix, gamma_kind, pow2, KeySrc{seq, 1, (n_bases + 31) / 32, (uint32_t)(2 * k)},
                      out, out_width, n, minimal, s, sms, rl);
}

// index(key) / index_no_remap(key) for one u64 key (ph_gpu_index_u64): the key is a launch
// parameter and one thread answers it (slot_of + remap_slot, index.hpp:91-100).
template <int G, bool POW2>
__global__ void __launch_bounds__(32) k_index_u64_one(const DevIndex ix, uint64_t key,
                                                      uint64_t* __restrict__ out, int minimal) {
    if (threadIdx.x) return;
    const uint64_t h = kC * (key ^ ix.seed);  // hash_int, hash.hpp:27
    uint64_t x;
    const uint32_t part = (uint32_t)mul32x64((uint32_t)ix.P, h, x);
    const uint32_t bucket = bucket_of<G>(x, (uint32_t)ix.B, ix.opt_table);
    const uint32_t pilot = ix.pilots[pilot_offset(ix, part, bucket)];
    uint64_t slot = (uint64_t)part * (uint32_t)ix.S + reduce<POW2>(ix, h ^ hash_pilot(ix, pilot));
    if (minimal && slot >= ix.n) slot = remap_get(ix, slot - ix.n);
    *out = slot;
}

cudaError_t launch_index_u64_one(const DevIndex& ix, int gamma_kind, bool pow2, uint64_t key,
                                 uint64_t* out, int minimal, cudaStream_t s) {
#define PH_CASE(G)                                                                         \
    case G:                                                                                \
        if (pow2) k_index_u64_one<G, true><<<1, 32, 0, s>>>(ix, key, out, minimal);       \
        else k_index_u64_one<G, false><<<1, 32, 0, s>>>(ix, key, out, minimal);           \
        break;
    switch (gamma_kind) {
        PH_CASE(0)
        PH_CASE(1)
        PH_CASE(2)
        PH_CASE(3)
        PH_CASE(4)
        default:
            return cudaErrorInvalidValue;
    }
#undef PH_CASE
    note_launch();
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Gather-only replay (measurement: bench.py's replay bound). The pilot reads of
// the query path at the index's true bucket addresses, in the order of `keys`, with the same
// key stream (8 B/key, evict_first) and the same pilot loads (evict_last) as pass B, and
// none of the slot arithmetic, remap or output: what those gathers alone cost. Over keys in
// query order it bounds the direct kernel; over keys sorted by partition group (pass B's
// order) it bounds pass B.
// ---------------------------------------------------------------------------
template <int G>
__global__ void __launch_bounds__(256, 4) k_gather_replay(const DevIndex ix,
                                                         const uint64_t* __restrict__ keys,
                                                         uint64_t n, uint32_t* __restrict__ sink) {
    constexpr int KPT = 8;
    const uint64_t pol_stream = policy_evict_first(), pol_keep = policy_evict_last();
    const uint32_t P32 = (uint32_t)ix.P, B32 = (uint32_t)ix.B;
    uint32_t acc = 0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * KPT;
    for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x * KPT; base < n; base += stride) {
        uint32_t pilot[KPT];
#pragma unroll
        for (int j = 0; j < KPT; j++) {
            const uint64_t i = base + (uint64_t)j * blockDim.x + threadIdx.x;
            const uint64_t h = kC * ((i < n ? ld_stream_u64(keys + i, pol_stream) : 0) ^ ix.seed);
            uint64_t x;
            const uint32_t part = (uint32_t)mul32x64(P32, h, x);
            const uint32_t bucket = bucket_of<G>(x, B32, ix.opt_table);
            pilot[j] = ld_gather_u8(ix.pilots + ((uint64_t)part * B32 + bucket), pol_keep);
        }
#pragma unroll
        for (int j = 0; j < KPT; j++) acc += pilot[j];
    }
    if (acc == 0xffffffffu) sink[0] = acc;  // (never: keeps the loads)
}

cudaError_t launch_gather_replay(const DevIndex& ix, int gamma_kind, const uint64_t* keys,
                                 uint64_t n, uint32_t* sink, cudaStream_t s, int sms) {
    if (n == 0) return cudaSuccess;
    const int grid = sms * 4;
    switch (gamma_kind) {
        case 0: k_gather_replay<0><<<grid, 256, 0, s>>>(ix, keys, n, sink); break;
        case 1: k_gather_replay<1><<<grid, 256, 0, s>>>(ix, keys, n, sink); break;
        case 2: k_gather_replay<2><<<grid, 256, 0, s>>>(ix, keys, n, sink); break;
        case 3: k_gather_replay<3><<<grid, 256, 0, s>>>(ix, keys, n, sink); break;
        case 4: k_gather_replay<4><<<grid, 256, 0, s>>>(ix, keys, n, sink); break;
        default: return cudaErrorInvalidValue;
    }
    note_launch();
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// index upload helper and the bijection verifier
// ---------------------------------------------------------------------------
// File-order pilots (P*B) -> hot-first layout, one part per block iteration.
__global__ void __launch_bounds__(256) k_relayout(const uint8_t* __restrict__ src,
                                                  uint8_t* __restrict__ dst, uint64_t P, uint64_t B,
                                                  uint64_t H) {
    for (uint64_t part = blockIdx.x; part < P; part += gridDim.x) {
        const uint8_t* s = src + part * B;
        uint8_t* hot = dst + part * H;
        uint8_t* cold = dst + P * H + part * (B - H);
        for (uint64_t b = threadIdx.x; b < B; b += blockDim.x) {
            const uint8_t v = s[b];
            if (b < H) hot[b] = v;
            else cold[b - H] = v;
        }
    }
}

cudaError_t launch_relayout(const uint8_t* src, uint8_t* dst, uint64_t P, uint64_t B, uint64_t H,
                            cudaStream_t s) {
    const uint64_t g = P < 65535 ? P : 65535;
    k_relayout<<<(unsigned)(g ? g : 1), 256, 0, s>>>(src, dst, P, B, H);
    return cudaGetLastError();
}

// verify_bijection (proj/tools/ptrhash.cpp:186-210) on the device: every output must be
// < n and hit exactly once. bits: ceil(n/32) zeroed words; bad[0] out-of-range, bad[1] dups.
template <class OutT>
__global__ void __launch_bounds__(256) k_verify(const OutT* __restrict__ out, uint64_t count,
                                                uint64_t n, unsigned int* bits,
                                                unsigned long long* bad) {
    unsigned long long oob = 0, dup = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t v = out[i];
        if (v >= n) {
            oob++;
            continue;
        }
        const unsigned int m = 1u << (v & 31);
        if (atomicOr(bits + (v >> 5), m) & m) dup++;
    }
    if (oob) atomicAdd(bad, oob);
    if (dup) atomicAdd(bad + 1, dup);
}

cudaError_t launch_verify(const void* out, int out_width, uint64_t count, uint64_t n,
                          unsigned int* bits, unsigned long long* bad, cudaStream_t s, int sms) {
    const int grid = sms * 8;
    if (out_width == 4)
        k_verify<uint32_t><<<grid, 256, 0, s>>>(static_cast<const uint32_t*>(out), count, n, bits, bad);
    else
        k_verify<uint64_t><<<grid, 256, 0, s>>>(static_cast<const uint64_t*>(out), count, n, bits, bad);
    note_launch();
    return cudaGetLastError();
}

}  // namespace phg
