// ph_partition.cu — the partitioned query path for DRAM-sized indexes.
//
// When the pilot array is far larger than what the L2 holds for random access (~64 MB),
// every direct query pays a DRAM row activation for its 1-byte pilot read (~57 G/s over
// 333 MB). This path turns those random DRAM reads into streaming passes plus L2-resident
// random reads. Keys are binned by hash group g = hi(G * h): group g's keys only use parts
// [gP/G, (g+1)P/G], a contiguous ~P*B/G-byte slice (32 MiB by default) of the pilots.
//
//   A  bin     per 4096-key tile (bulk-copied into shared memory): ranks by group with
//              shared-memory atomics, one global atomicAdd per (tile, group) reserves a run
//              in that group's region, and each run leaves shared memory as bulk stores:
//              entry = (key, position in the tile as u16); run (offset, length) ->
//              runoff/runcnt[tile][g].
//   B  query   one persistent kernel; CTAs claim chunks of the group regions in order from
//              a global counter, so the chunks in flight stay within one or two slices,
//              which stay L2-resident (evict_last). Full query arithmetic incl. remap_slot;
//              answers into slots[] at the same entry index.
//   C  unbin   per tile: the G runs' (position, slot) pairs are bulk-loaded, scattered into
//              a shared-memory tile and written to out[] with one bulk store.
//
// Group regions have a fixed capacity (n/G plus 16 sigma plus a tile); a run that does not
// fit goes to a spill region sized for the worst case (any distribution of queries, e.g.
// one key repeated n times, is answered correctly; only the L2 locality of pass B is lost).
// Unused region tails hold stale entries that pass B answers harmlessly and pass C never
// reads. Results are identical to the direct kernel: pass B runs the same arithmetic.
//
// DRAM bytes per query: A 8 (key) + 10 (entry), B 8 + 4 (u32 slot), C 6 + 4 = 40 B, all
// streamed, against the direct kernel's 12 B streamed + one DRAM row activation per query.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>

#include "ph_device.cuh"
#include "ph_kernels.h"
#include "ph_nvtx.h"

namespace phg {

// Checked builds (-DPH_CHECKS, tools/checked_run.py; compute-sanitizer is closed on this GPU
// pool): every shared-memory staging index, bulk-copy range and scatter position of passes
// A-C is bounds-checked on the device, and a canary band after the scratch is verified.
// Violations are counted (no trap), read back with ph_gpu_check_errors.
#ifdef PH_CHECKS
struct ChkBounds {
    uint64_t nent;       // entries in bins / bpos / slots
    uint64_t n;          // keys (windows)
    uint64_t in_words;   // words readable at `keys` (u64 keys: n; k-mers: sequence words)
    uint64_t ntiles;
};
__device__ ChkBounds g_chk_b;
__device__ unsigned long long g_chk[2];  // [0] violations, [1] source line of the first
#define PH_CHECK(c)                                                                   \
    do {                                                                              \
        if (!(c) && atomicAdd(&g_chk[0], 1ull) == 0) g_chk[1] = __LINE__;            \
    } while (0)
#else
#define PH_CHECK(c) \
    do {            \
    } while (0)
#endif

#ifndef PH_TILE_KEYS
#define PH_TILE_KEYS 4096
#endif
constexpr int kBinThreads = 256;
constexpr uint32_t kTileKeys = PH_TILE_KEYS;  // keys per tile (positions are u16)
constexpr int kBinPerThread = kTileKeys / kBinThreads;
constexpr int kBinCtas = 4;    // CTAs per SM (registers: 64 per thread)
constexpr int kMaxGroups = 64;
constexpr uint16_t kPadPos = 0xffff;  // position of a run's padding entry (never a tile position)
// ctrl[]: per-group cursors [0, kMaxGroups), spill cursor, pass B's chunk counter
constexpr int kCtrlSpill = kMaxGroups;
constexpr int kCtrlWork = kMaxGroups + 1;
constexpr int kCtrlWords = kMaxGroups + 2;

// Group of a key: g = hi32(G * hi32(h)) for the hash h = C * (key ^ seed) (hash.hpp:27).
// Monotone in h like part = hi(P * h) (bucket_fn.hpp:66-72), so each group's keys use a
// contiguous range of parts. Only the high word of h is formed (3 multiplies).
__device__ __forceinline__ uint32_t group_of(uint64_t key, uint64_t seed, uint32_t G) {
    const uint64_t x = key ^ seed;
    const uint32_t xl = (uint32_t)x, xh = (uint32_t)(x >> 32);
    const uint32_t hh = __umulhi(xl, (uint32_t)kC) + xl * (uint32_t)(kC >> 32) + xh * (uint32_t)kC;
    return __umulhi(hh, G);
}

// k-mer of window i (same layout and arithmetic as kmer_at in ph_query.cu).
__device__ __forceinline__ uint64_t part_kmer(const uint64_t* __restrict__ seq, uint64_t nwords,
                                              uint64_t i, uint32_t kbits) {
    const uint64_t a = i >> 5;
    const uint32_t o = (uint32_t)(i & 31) * 2;
    const uint64_t wa = __ldg(seq + a);
    const uint64_t wb = (o && a + 1 < nwords) ? __ldg(seq + a + 1) : 0;
    const uint64_t top = o ? (wa << o) | (wb >> (64 - o)) : wa;
    return kbits == 64 ? top : top >> (64 - kbits);
}

// Reserves a run for c entries of group g: c rounded up to a multiple of 8 entries, so
// every run starts 64-B aligned in bins[] and 16-B aligned in bpos[] / slots[] (the bulk
// copies of passes A and C need that). Group regions hold `cap` entries; a run that does
// not fit goes to the spill region after them.
__device__ __forceinline__ uint64_t reserve_run(unsigned long long* ctrl, uint32_t g, uint32_t c,
                                                uint32_t G, uint64_t cap) {
    if (!c) return 0;
    const unsigned long long c8 = (c + 7u) & ~7u;

    const uint64_t off = atomicAdd(ctrl + g, c8);
    return off + c8 <= cap ? g * cap + off : G * cap + atomicAdd(ctrl + kCtrlSpill, c8);
}

__device__ __forceinline__ void st_cs_u64(uint64_t* p, uint64_t v) {
    asm volatile("st.global.cs.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_cs_u16(uint16_t* p, uint16_t v) {
    asm volatile("st.global.cs.u16 [%0], %1;" ::"l"(p), "h"(v) : "memory");
}

// Pass A. Per tile: per-group counts and ranks with shared-memory atomics (the order
// within a run does not matter: each entry carries its tile position), run reservation by
// warp 0 (one global atomicAdd per group), staging in group order, then every thread
// writes 16 staged entries (balanced, coalesced within runs). The next tile's keys are
// loaded before the run writes. 4 CTAs per SM overlap one another's barrier phases.
template <int SRC>
__global__ void __launch_bounds__(kBinThreads, kBinCtas) k_bin(
    const uint64_t* __restrict__ keys, uint64_t n, uint64_t seq_words, uint32_t kbits,
    uint64_t seed, uint32_t G, uint64_t cap, unsigned long long* __restrict__ ctrl,
    uint64_t* __restrict__ runoff, uint16_t* __restrict__ runcnt, uint64_t* __restrict__ bins,
    uint16_t* __restrict__ bpos) {
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t* sk = reinterpret_cast<uint64_t*>(smem);
    uint32_t* spg = reinterpret_cast<uint32_t*>(sk + kTileKeys);  // tile position | group << 16
    __shared__ uint32_t cnt[2][kMaxGroups];
    __shared__ uint32_t lbase[kMaxGroups];
    __shared__ uint64_t delta[kMaxGroups];  // run offset - staged offset
    const unsigned tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t ntiles = (n + kTileKeys - 1) / kTileKeys;
    uint64_t k[kBinPerThread];
    auto load = [&](uint64_t t) {
        const uint64_t t0 = t * kTileKeys;
        const uint32_t valid = (uint32_t)(n - t0 < kTileKeys ? n - t0 : kTileKeys);
#pragma unroll
        for (int j = 0; j < kBinPerThread; j++) {
            const uint32_t e = (uint32_t)j * kBinThreads + tid;
            if (SRC == 1)
                k[j] = e < valid ? part_kmer(keys, seq_words, t0 + e, kbits) : 0;
            else
                k[j] = e < valid ? __ldcs(keys + t0 + e) : 0;
        }
    };
    if (tid < kMaxGroups) cnt[0][tid] = 0;
    uint64_t t = blockIdx.x;
    if (t < ntiles) load(t);
    __syncthreads();
    for (int par = 0; t < ntiles; t += gridDim.x, par ^= 1) {
        const uint64_t t0 = t * kTileKeys;
        const uint32_t valid = (uint32_t)(n - t0 < kTileKeys ? n - t0 : kTileKeys);
        uint32_t* c_ = cnt[par];
        uint32_t gr[kBinPerThread];  // group << 16 | rank
#pragma unroll
        for (int j = 0; j < kBinPerThread; j++) {
            if ((uint32_t)j * kBinThreads + tid < valid) {
                const uint32_t g = group_of(k[j], seed, G);
                gr[j] = g << 16 | atomicAdd(&c_[g], 1u);
            }
        }
        __syncthreads();
        if (tid < kMaxGroups) cnt[par ^ 1][tid] = 0;  // next tile's counters
        uint32_t c0 = 0, c1 = 0;
        if (warp == 0) {  // lane owns groups 2*lane and 2*lane+1
            const uint32_t g0 = 2 * lane;
            c0 = g0 < G ? c_[g0] : 0;
            c1 = g0 + 1 < G ? c_[g0 + 1] : 0;
            uint32_t x = c0 + c1;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(kFull, x, o);
                if (lane >= (unsigned)o) x += y;
            }
            x -= c0 + c1;
            lbase[g0] = x;
            lbase[g0 + 1] = x + c0;
        }
        __syncthreads();
        if (warp == 0) {  // run reservations; their latency overlaps the other warps' staging
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const uint32_t g = 2 * lane + h, c = h ? c1 : c0;
                if (g < G) {
                    const uint64_t off = reserve_run(ctrl, g, c, G, cap);
                    for (uint32_t i = c; i < ((c + 7u) & ~7u); i++) bpos[off + i] = kPadPos;
                    delta[g] = off - lbase[g];
                    runoff[t * G + g] = off;
                    runcnt[t * G + g] = (uint16_t)c;
                }
            }
        }
#pragma unroll
        for (int j = 0; j < kBinPerThread; j++) {
            const uint32_t pos = (uint32_t)j * kBinThreads + tid;
            if (pos < valid) {
                const uint32_t g = gr[j] >> 16;
                const uint32_t e = lbase[g] + (gr[j] & 0xffffu);
                sk[e] = k[j];
                spg[e] = pos | g << 16;
            }
        }
        __syncthreads();
        if (t + gridDim.x < ntiles) load(t + gridDim.x);
#pragma unroll 4
        for (int j = 0; j < kBinPerThread; j++) {
            const uint32_t e = (uint32_t)j * kBinThreads + tid;
            if (e < valid) {
                const uint32_t pg = spg[e];
                const uint64_t dst = delta[pg >> 16] + e;
                st_cs_u64(bins + dst, sk[e]);
                st_cs_u16(bpos + dst, (uint16_t)pg);
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// Bulk-copy (TMA engine, cp.async.bulk) variants of passes A and C: tiles of keys arrive in
// shared memory by bulk loads completing on an mbarrier (double-buffered, issued two tiles
// ahead), and every staged run leaves with one bulk store per array. Threads only rank,
// place and scatter in shared memory. Used when the key array is 16-B aligned.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// global -> shared, completes `bytes` on bar (16-B aligned, multiple of 16)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}
// shared -> global, bulk-group completion (16-B aligned, multiple of 16)
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes, uint64_t pol) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(
                     dst),
                 "r"(smem_u32(src)), "r"(bytes), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
// at most one bulk group (the most recent) may still be reading shared memory
__device__ __forceinline__ void bulk_wait_read1() {
    asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

constexpr uint32_t kStageEntries = kTileKeys + 7 * kMaxGroups;  // runs padded to 8 entries
constexpr int kTmaGroups = 32;  // pass A's bulk-copy variant: G <= 32 (lane = group)

constexpr uint32_t kBinTmaStage = kTileKeys + 8 * kTmaGroups;  // (a multiple of 8)
#ifndef PH_BIN_TMA_THREADS
#define PH_BIN_TMA_THREADS 512
#endif
constexpr int kBinTmaThreads = PH_BIN_TMA_THREADS;
// input buffers: a u64 key tile, or (k-mers) the tile's kSeqWords packed words
template <int SRC>
constexpr uint32_t bin_in_words() { return SRC == 1 ? (kTileKeys / 32 + 2 + 1) & ~1u : kTileKeys; }
template <int SRC>
constexpr size_t bin_tma_smem() { return 2 * bin_in_words<SRC>() * 8 + kBinTmaStage * (8 + 2); }
#ifndef PH_BIN_KMER_CTAS
#define PH_BIN_KMER_CTAS 3  // k-mer pass A CTAs per SM (2 KB input buffers; 3 vs 2: 3.57 vs 3.83 ms at config 5)
#endif

// Pass A, bulk-copy variant (u64 keys, 16-B aligned key array).
// SRC = 1: keys are the k-mers of a packed sequence (seq_words, kbits): a tile's windows
// need its kSeqWords packed words (0.25 B per key), which arrive by bulk load like u64 key
// tiles, and each window is extracted from shared memory.
constexpr uint32_t kSeqWords = kTileKeys / 32 + 2;  // 130: 16-B multiple for 4096-key tiles
template <int THREADS, int SRC>
__global__ void __launch_bounds__(THREADS, SRC == 1 ? PH_BIN_KMER_CTAS : 2) k_bin_tma(
    const uint64_t* __restrict__ keys, uint64_t n, uint64_t seq_words, uint32_t kbits,
    uint64_t seed, uint32_t G, uint64_t cap,
    unsigned long long* __restrict__ ctrl, uint64_t* __restrict__ runoff,
    uint16_t* __restrict__ runcnt, uint64_t* __restrict__ bins, uint16_t* __restrict__ bpos) {
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t* in = reinterpret_cast<uint64_t*>(smem);  // [2][kTileKeys]
    constexpr uint32_t IW = bin_in_words<SRC>();         // words per input buffer
    uint64_t* sk = in + 2 * IW;                          // staged keys, runs 8-aligned
    uint16_t* sp = reinterpret_cast<uint16_t*>(sk + kBinTmaStage);
    __shared__ __align__(8) uint64_t bar[2];
    __shared__ uint32_t cnt[2][kTmaGroups];
    __shared__ uint32_t lb8[kTmaGroups];  // staging bases (the k-mer variant's shared scan)
    constexpr int PER = kTileKeys / THREADS;
    const unsigned tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t ntiles = (n + kTileKeys - 1) / kTileKeys;
    // tiles that arrive by bulk load: whole u64 key tiles, or (k-mers) tiles whose
    // kSeqWords words all lie inside the sequence
    const bool aligned = (reinterpret_cast<uintptr_t>(keys) & 15) == 0;
    const uint64_t nfull =
        !aligned ? 0
        : SRC == 0 ? n / kTileKeys
                   : (seq_words >= kSeqWords
                          ? min((seq_words - kSeqWords) / (kTileKeys / 32) + 1, ntiles)
                          : 0);
    auto bulk = [&](uint64_t t) { return t < nfull; };
    const uint64_t pol = policy_evict_first();
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
    }
    if (tid < kTmaGroups) cnt[0][tid] = 0;
    __syncthreads();
    auto issue = [&](uint64_t t, int b) {  // thread 0: bulk-load tile t's input into buffer b
        constexpr uint32_t bytes = SRC == 1 ? kSeqWords * 8 : kTileKeys * 8;
#ifdef PH_CHECKS
        PH_CHECK(t * (SRC == 1 ? kTileKeys / 32 : kTileKeys) + bytes / 8 <= g_chk_b.in_words);
#endif
        mbar_expect_tx(&bar[b], bytes);
        bulk_g2s(in + b * IW, keys + t * (SRC == 1 ? kTileKeys / 32 : kTileKeys), bytes,
                 &bar[b], pol);
    };
    if (tid == 0) {
        if (bulk(blockIdx.x)) issue(blockIdx.x, 0);
        if (bulk(blockIdx.x + gridDim.x)) issue(blockIdx.x + gridDim.x, 1);
    }
    uint32_t it = 0;
    for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x, it++) {
        const int b = it & 1;
        const uint64_t t0 = t * kTileKeys;
        const uint32_t valid = (uint32_t)(n - t0 < kTileKeys ? n - t0 : kTileKeys);
        uint64_t k[PER];
        if (SRC == 1) {
            // k-mers: the tile's packed words (each serves 32 consecutive windows) sit in
            // shared memory -- bulk-loaded ahead, or (last tiles) loaded here -- and every
            // window is extracted from there (kmer_at's layout)
            const uint64_t w0 = t0 >> 5;
            uint64_t* wv = in + b * IW;
            if (bulk(t)) {
                mbar_wait(&bar[b], (it >> 1) & 1);
            } else {
                const uint64_t left = seq_words - w0;
                const uint32_t nw = (uint32_t)(left < kSeqWords ? left : kSeqWords);
                for (uint32_t q = tid; q < nw; q += THREADS) wv[q] = __ldg(keys + w0 + q);
                __syncthreads();
            }
#pragma unroll
            for (int j = 0; j < PER; j++) {
                const uint32_t e = (uint32_t)j * THREADS + tid;
                const uint64_t i = t0 + e;
                const uint32_t a = (uint32_t)((i >> 5) - w0), o = (uint32_t)(i & 31) * 2;
                const uint64_t wa = wv[a];
                const uint64_t wb = (o && w0 + a + 1 < seq_words) ? wv[a + 1] : 0;
                const uint64_t top = o ? (wa << o) | (wb >> (64 - o)) : wa;
                k[j] = e < valid ? (kbits == 64 ? top : top >> (64 - kbits)) : 0;
            }
        } else if (bulk(t)) {
            mbar_wait(&bar[b], (it >> 1) & 1);
#pragma unroll
            for (int j = 0; j < PER; j++) k[j] = in[b * IW + j * THREADS + tid];
        } else {
#pragma unroll
            for (int j = 0; j < PER; j++) {
                const uint32_t e = (uint32_t)j * THREADS + tid;
                k[j] = e < valid ? __ldcs(keys + t0 + e) : 0;
            }
        }
        uint32_t* c_ = cnt[b];
        // TWO: two CTA barriers per tile (u64 keys). Warp 0 waits for the previous tile's run
        // stores to finish reading the staging buffer while the other warps rank, and every
        // warp scans the group counts itself. Otherwise (k-mers, whose ranking is too short
        // to hide that wait) warp 0 waits after barrier #1 and publishes the scan behind a
        // second barrier (u64: 3.18 -> 3.07 ms at config 3; k-mers: 3.58 vs 3.79 ms).
        constexpr bool TWO = SRC == 0;
        if (TWO && warp == 0) bulk_wait_read();
        uint32_t gr[PER];  // group << 16 | rank
#pragma unroll
        for (int j = 0; j < PER; j++) {
            gr[j] = 0;
            if ((uint32_t)j * THREADS + tid < valid) {
                const uint32_t g = group_of(k[j], seed, G);
                gr[j] = g << 16 | atomicAdd(&c_[g], 1u);
            }
        }
        __syncthreads();  // #1: buffer b consumed, counts final (TWO: staging free)
        if (tid == 0 && bulk(t + 2 * (uint64_t)gridDim.x)) issue(t + 2 * (uint64_t)gridDim.x, b);
        if (tid < kTmaGroups) cnt[b ^ 1][tid] = 0;  // next tile's counters
        // lane g: group g's count; warp 0 reserves the runs (one global atomicAdd per group,
        // its latency overlapping the scan and the staging)
        uint32_t c = 0, lb = 0;
        unsigned long long a = 0;
        if (TWO || warp == 0) {
            c = lane < G ? c_[lane] : 0;
            if (warp == 0 && c) a = atomicAdd(ctrl + lane, (unsigned long long)((c + 7) & ~7u));
            if (!TWO) bulk_wait_read();  // the previous tile's run stores have read the staging
            const uint32_t p8 = (c + 7) & ~7u;
            uint32_t x = p8;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(kFull, x, o);
                if (lane >= (unsigned)o) x += y;
            }
            lb = x - p8;  // this lane's group's staging base
            if (!TWO) lb8[lane] = lb;
        }
        if (!TWO) __syncthreads();  // #2: staging free, lb8 final
#pragma unroll
        for (int j = 0; j < PER; j++) {
            const uint32_t pos = (uint32_t)j * THREADS + tid;
            const uint32_t base = TWO ? __shfl_sync(kFull, lb, gr[j] >> 16) : lb8[gr[j] >> 16];
            const uint32_t e = base + (gr[j] & 0xffffu);
            if (pos < valid) {
                PH_CHECK(e < kBinTmaStage && (gr[j] >> 16) < G);
                sk[e] = k[j];
                sp[e] = (uint16_t)pos;
            }
        }
        uint64_t off = 0;
        if (warp == 0 && lane < G) {  // consume the reservation (spill if the region is full)
            const unsigned long long c8 = (c + 7u) & ~7u;
            for (uint32_t i = c; i < c8; i++) sp[lb + i] = kPadPos;  // padding entries
            off = !c ? 0 : a + c8 <= cap ? lane * cap + a : G * cap + atomicAdd(ctrl + kCtrlSpill, c8);
            runoff[t * G + lane] = off;
            runcnt[t * G + lane] = (uint16_t)c;
        }
        fence_async_smem();
        __syncthreads();  // staged; run offsets known
        if (warp == 0) {  // lane issues the bulk stores of its group's run
            const uint32_t p8 = (c + 7) & ~7u;
            if (lane < G && c) {
#ifdef PH_CHECKS
                PH_CHECK(lb + p8 <= kBinTmaStage && off + p8 <= g_chk_b.nent && (off & 7) == 0);
#endif
                bulk_s2g(bins + off, sk + lb, p8 * 8, pol);
                bulk_s2g(bpos + off, sp + lb, p8 * 2, pol);
            }
            bulk_commit();
        }
    }
    if (warp == 0) bulk_wait_all();
}

// Pass C, bulk-copy variant: the tile's runs (8-entry aligned) arrive by bulk loads two
// tiles ahead (double-buffered), are scattered by position into the output tile in shared
// memory, and the output tile leaves with one bulk store when `out` is 16-B aligned. Warp 0
// loads the run table of the tile it will issue next at the top of each iteration, so the
// issue at the bottom does not wait on global loads while the other warps wait for it.
template <class OutT>
struct UnbinTma {
    static constexpr size_t kIn = (size_t)kStageEntries * (sizeof(OutT) + 2);  // one buffer
    static constexpr size_t kSmem = 2 * kIn + (size_t)kTileKeys * sizeof(OutT);
};

template <class OutT>
__global__ void __launch_bounds__(kBinThreads) k_unbin_tma(
    uint64_t n, uint32_t G, const uint64_t* __restrict__ runoff,
    const uint16_t* __restrict__ runcnt, const uint16_t* __restrict__ bpos,
    const OutT* __restrict__ slots, OutT* __restrict__ out) {
    extern __shared__ __align__(128) uint8_t smem[];
    OutT* stage = reinterpret_cast<OutT*>(smem + 2 * UnbinTma<OutT>::kIn);
    __shared__ __align__(8) uint64_t bar[2];
    __shared__ uint32_t mtot[2];             // per buffer: staged entries (runs padded to 8)
    const unsigned tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t ntiles = (n + kTileKeys - 1) / kTileKeys;
    const bool vec = (reinterpret_cast<uintptr_t>(out) & 15) == 0;
    const uint64_t pol = policy_evict_first();
    auto bufs = [&](int b, OutT*& sv, uint16_t*& pv) {
        sv = reinterpret_cast<OutT*>(smem + b * UnbinTma<OutT>::kIn);
        pv = reinterpret_cast<uint16_t*>(sv + kStageEntries);
    };
    struct Meta {  // warp 0, lane l: the runs of groups 2l and 2l+1
        uint32_t c0, c1;
        uint64_t o0, o1;
    };
    auto meta = [&](uint64_t t) {
        Meta m{0, 0, 0, 0};
        const uint32_t g0 = 2 * lane;
        if (t < ntiles) {
            if (g0 < G) m.c0 = __ldg(runcnt + t * G + g0), m.o0 = __ldg(runoff + t * G + g0);
            if (g0 + 1 < G) m.c1 = __ldg(runcnt + t * G + g0 + 1), m.o1 = __ldg(runoff + t * G + g0 + 1);
        }
        return m;
    };
    // warp 0: bulk-load a tile's runs (described by m) into buffer b
    auto issue = [&](const Meta& m, int b) {
        const uint32_t p0 = (m.c0 + 7) & ~7u, p1 = (m.c1 + 7) & ~7u;
        uint32_t x = p0 + p1;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, x, o);
            if (lane >= (unsigned)o) x += y;
        }
        const uint32_t total = __shfl_sync(kFull, x, 31);
        x -= p0 + p1;
        if (lane == 0) {
            mtot[b] = total;
            mbar_expect_tx(&bar[b], total * (uint32_t)(sizeof(OutT) + 2));
        }
        __syncwarp();
        OutT* sv;
        uint16_t* pv;
        bufs(b, sv, pv);
#ifdef PH_CHECKS
        PH_CHECK(x + p0 + p1 <= kStageEntries && total <= kStageEntries);
        PH_CHECK((!p0 || m.o0 + p0 <= g_chk_b.nent) && (!p1 || m.o1 + p1 <= g_chk_b.nent));
#endif
        if (p0) {
            bulk_g2s(sv + x, slots + m.o0, p0 * (uint32_t)sizeof(OutT), &bar[b], pol);
            bulk_g2s(pv + x, bpos + m.o0, p0 * 2, &bar[b], pol);
        }
        if (p1) {
            bulk_g2s(sv + x + p0, slots + m.o1, p1 * (uint32_t)sizeof(OutT), &bar[b], pol);
            bulk_g2s(pv + x + p0, bpos + m.o1, p1 * 2, &bar[b], pol);
        }
    };
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (warp == 0) {
        if (blockIdx.x < ntiles) issue(meta(blockIdx.x), 0);
        if (blockIdx.x + gridDim.x < ntiles) issue(meta(blockIdx.x + gridDim.x), 1);
    }
    uint32_t it = 0;
    for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x, it++) {
        const int b = it & 1;
        const uint64_t t0 = t * kTileKeys;
        const uint32_t valid = (uint32_t)(n - t0 < kTileKeys ? n - t0 : kTileKeys);
        const uint64_t tn = t + 2 * (uint64_t)gridDim.x;  // the tile buffer b serves next
        Meta mn{0, 0, 0, 0};
        if (warp == 0) mn = meta(tn);
        mbar_wait(&bar[b], (it >> 1) & 1);
        if (tid == 0) bulk_wait_read();  // the previous output tile has left `stage`
        __syncthreads();
        OutT* sv;
        uint16_t* pv;
        bufs(b, sv, pv);
        // every staged entry in parallel; padding entries carry position kPadPos
        const uint32_t total = mtot[b];
#pragma unroll 4
        for (uint32_t e = tid; e < total; e += kBinThreads) {
            const uint16_t p = pv[e];
            PH_CHECK(p == kPadPos || p < valid);
            if (p != kPadPos) stage[p] = sv[e];
        }
        fence_async_smem();
        __syncthreads();
        if (vec && valid == kTileKeys) {
            if (tid == 0) {
                bulk_s2g(out + t0, stage, kTileKeys * (uint32_t)sizeof(OutT), pol);
                bulk_commit();
            }
        } else {
            for (uint32_t e = tid; e < valid; e += kBinThreads) st_stream(out + t0 + e, stage[e]);
        }
        if (warp == 0 && tn < ntiles) issue(mn, b);
    }
    if (tid == 0) bulk_wait_all();
}

// Pass B: the query arithmetic, remap_slot included, over the group regions (region r < G:
// group r, r == G: the spill); slots[] gets each entry's answer at the same entry index.
// CTAs claim batches of 2048-entry chunks in order from a global counter, so the chunks in
// flight always form one contiguous window (one or two regions): the current pilot slice
// stays L2-resident. (Measured and not kept: each chunk's entries bulk-copied into shared
// memory a chunk ahead by a producer thread, 5.40 vs 5.22 ms at config 3.)
constexpr int kQThreads = 256;
#ifndef PH_QB_PER
#define PH_QB_PER 8
#endif
constexpr int kQPer = PH_QB_PER;                      // keys per thread (pairs)
constexpr uint32_t kQChunk = kQThreads * kQPer;       // 2048 entries per chunk
#ifndef PH_QB_MINB
#define PH_QB_MINB 4
#endif
#ifndef PH_QB_SEPARATE
#define PH_QB_SEPARATE 1  // all buckets first, then the gathers back to back (5.10 vs 5.38 ms interleaved)
#endif
#ifndef PH_QB_CLAIM
#define PH_QB_CLAIM 8  // chunks per claim, one CTA barrier per claim (1, 2, 4, 8, 16, 32 swept: 8-16 best, ~1 %)
#endif

template <int G, bool POW2, class OutT, int MF>
__global__ void __launch_bounds__(kQThreads, PH_QB_MINB) k_query_regions(
    const DevIndex ix, uint32_t NG, uint64_t cap, unsigned long long* __restrict__ ctrl,
    const uint64_t* __restrict__ bins, OutT* __restrict__ slots, int minimal) {
    __shared__ uint64_t cstart[kMaxGroups + 2];  // first chunk of each region
    __shared__ uint64_t rend[kMaxGroups + 1];    // entry end of each region
    __shared__ uint64_t claim[2];
    const unsigned tid = threadIdx.x;
    if (tid == 0) {
        uint64_t c = 0;
        for (uint32_t r = 0; r <= NG; r++) {
            const uint64_t len = r < NG ? min((uint64_t)ctrl[r], cap) : (uint64_t)ctrl[kCtrlSpill];
            cstart[r] = c;
            rend[r] = (uint64_t)r * cap + len;
            c += (len + kQChunk - 1) / kQChunk;
        }
        cstart[NG + 1] = c;
        claim[0] = atomicAdd(ctrl + kCtrlWork, 1ull);
    }
    __syncthreads();
    const uint64_t nchunks = cstart[NG + 1];
    const uint64_t pol_stream = policy_evict_first();
    const uint64_t pol_keep = ix.pilot_evict_normal ? policy_evict_normal() : policy_evict_last();
    const uint32_t P32 = (uint32_t)ix.P, B32 = (uint32_t)ix.B, S32 = (uint32_t)ix.S;
    uint32_t r = 0;
    for (int k = 0;; k ^= 1) {
        const uint64_t c0 = claim[k] * PH_QB_CLAIM;  // a batch of PH_QB_CLAIM chunks
        if (c0 >= nchunks) break;
        if (tid == 0) claim[k ^ 1] = atomicAdd(ctrl + kCtrlWork, 1ull);  // next, in flight
      for (uint64_t c = c0; c < c0 + PH_QB_CLAIM && c < nchunks; c++) {
        while (c >= cstart[r + 1]) r++;
        const uint64_t e0 = (uint64_t)r * cap + (c - cstart[r]) * kQChunk;
        const uint64_t end = rend[r];  // region lengths are multiples of 8 entries
#ifdef PH_CHECKS
        PH_CHECK(end <= g_chk_b.nent && (end & 7) == 0 && e0 < end);
#endif
        uint64_t h[kQPer];
#pragma unroll
        for (int q = 0; q < kQPer / 2; q++) {
            const uint64_t e = e0 + ((uint64_t)q * kQThreads + tid) * 2;
            h[2 * q] = h[2 * q + 1] = 0;
            if (e < end)
                asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u64 {%0,%1}, [%2], %3;"
                    : "=l"(h[2 * q]), "=l"(h[2 * q + 1])
                    : "l"(bins + e), "l"(pol_stream));
        }
        uint32_t part[kQPer], pilot[kQPer];
#pragma unroll
        for (int j = 0; j < kQPer; j++) {
            h[j] = kC * (h[j] ^ ix.seed);  // hash_int, hash.hpp:27
            uint64_t x;
            part[j] = (uint32_t)mul32x64(P32, h[j], x);  // part_and_bucket, bucket_fn.hpp:66-72
            const uint32_t bucket = bucket_of<G>(x, B32, ix.opt_table);
#if PH_QB_SEPARATE
            pilot[j] = bucket;
        }
#pragma unroll
        for (int j = 0; j < kQPer; j++) {  // the gathers back to back (pilot[j] = bucket)
            pilot[j] = ld_gather_u8(ix.pilots + ((uint64_t)part[j] * B32 + pilot[j]), pol_keep);
#else
            pilot[j] = ld_gather_u8(ix.pilots + ((uint64_t)part[j] * B32 + bucket), pol_keep);
#endif
        }
        uint64_t slot[kQPer];
        bool need[kQPer];
#pragma unroll
        for (int j = 0; j < kQPer; j++) {  // slot_of, index.hpp:91-96
            slot[j] = (uint64_t)part[j] * S32 + reduce<POW2, MF>(ix, h[j] ^ hash_pilot(ix, pilot[j]));
            const uint64_t e = e0 + ((uint64_t)(j >> 1) * kQThreads + tid) * 2 + (j & 1);
            need[j] = minimal && slot[j] >= ix.n && e < end;
        }
        // remap_slot (index.hpp:98-100) for the ~1 % of slots >= n: ranked across the warp
        // with ballots, one convergent round of CacheLineEF decodes (L2-resident table)
        if (minimal) remap_tile<kQPer, OutT>(ix, need, slot);
#pragma unroll
        for (int q = 0; q < kQPer / 2; q++) {
            const uint64_t e = e0 + ((uint64_t)q * kQThreads + tid) * 2;
            if (e < end) {
                if constexpr (sizeof(OutT) == 4)
                    asm volatile("st.global.cs.v2.u32 [%0], {%1,%2};" ::"l"(slots + e),
                                 "r"((uint32_t)slot[2 * q]), "r"((uint32_t)slot[2 * q + 1])
                                 : "memory");
                else
                    asm volatile("st.global.cs.v2.u64 [%0], {%1,%2};" ::"l"(slots + e),
                                 "l"(slot[2 * q]), "l"(slot[2 * q + 1])
                                 : "memory");
            }
        }
      }
        __syncthreads();  // claim[k ^ 1] visible; claim[k] free for reuse
    }
}

template <class OutT>
static cudaError_t launch_regions(const DevIndex& ix, int gamma_kind, bool pow2, uint32_t G,
                                  uint64_t cap, uint64_t nent, unsigned long long* ctrl,
                                  const uint64_t* bins, OutT* slots, int minimal, cudaStream_t s,
                                  int sms, int per_sm) {
    const uint64_t chunks_max = nent / kQChunk + G + 2;
    const int grid = (int)std::min<uint64_t>(chunks_max, (uint64_t)sms * per_sm);
#define PH_CASE(GK)                                                                              \
    case GK:                                                                                     \
        if (pow2) k_query_regions<GK, true, OutT, 0><<<grid, kQThreads, 0, s>>>(ix, G, cap, ctrl, bins, slots, minimal); \
        else if (ix.mod_fast_ok) k_query_regions<GK, false, OutT, 1><<<grid, kQThreads, 0, s>>>(ix, G, cap, ctrl, bins, slots, minimal); \
        else k_query_regions<GK, false, OutT, 0><<<grid, kQThreads, 0, s>>>(ix, G, cap, ctrl, bins, slots, minimal);    \
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
#ifdef PH_CHECKS
constexpr uint64_t kCanaryBytes = 4096;
__global__ void k_canary_check(const uint32_t* p, uint32_t words) {
    for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) PH_CHECK(p[i] == 0xA5A5A5A5u);
}
#endif
namespace {
struct Layout {
    uint64_t cap, ntiles, nent;
    uint64_t o_runoff, o_runcnt, o_bins, o_bpos, o_slots, total;
};
Layout layout(uint64_t n, uint32_t G, int out_width) {
    auto al = [](uint64_t b) { return (b + 255) & ~uint64_t{255}; };
    Layout L;
    const uint64_t per = (n + G - 1) / G;
    L.ntiles = (n + kTileKeys - 1) / kTileKeys;
    // n/G + 16 sigma + one tile + up to 7 padding entries per tile (8-entry aligned runs)
    L.cap = per + 16 * (uint64_t)std::ceil(std::sqrt((double)per)) + kTileKeys + 7 * L.ntiles;
    L.cap = (L.cap + 255) & ~uint64_t{255};
    // spill: worst case every entry, each run padded by up to 7
    L.nent = G * L.cap + n + 7 * std::min<uint64_t>(n, L.ntiles * G);
    uint64_t o = al(kCtrlWords * 8);
    L.o_runoff = o;
    o += al(L.ntiles * G * 8);
    L.o_runcnt = o;
    o += al(L.ntiles * G * 2);
    L.o_bins = o;
    o += al(L.nent * 8);
    L.o_bpos = o;
    o += al(L.nent * 2);
    L.o_slots = o;
    o += al(L.nent * (uint64_t)out_width);
#ifdef PH_CHECKS
    o += kCanaryBytes;  // canary band after the scratch (checked builds)
#endif
    L.total = o;
    return L;
}
}  // namespace

// Optional per-pass timing (ph_gpu_set_pass_timing / ph_gpu_pass_times): cudaEvents on the
// call's stream around passes A, B and C of up to kTimedCalls calls. A profiling aid for
// bench.py's per-pass roofline; one host thread at a time.
namespace {
constexpr int kTimedCalls = 256;
struct PassTiming {
    bool on = false;
    int calls = 0;
    cudaEvent_t ev[kTimedCalls][4] = {};
} g_pt;
void pt_record(int k, cudaStream_t s) {
    if (!g_pt.on || g_pt.calls >= kTimedCalls) return;
    cudaEvent_t& e = g_pt.ev[g_pt.calls][k];
    if (!e) cudaEventCreate(&e);
    cudaEventRecord(e, s);
    if (k == 3) g_pt.calls++;
}
}  // namespace

void set_pass_timing(bool on) {
    g_pt.on = on;
    g_pt.calls = 0;
}

int pass_times(double* ms_sums, int* calls) {
    ms_sums[0] = ms_sums[1] = ms_sums[2] = 0;
    for (int c = 0; c < g_pt.calls; c++) {
        cudaEvent_t* e = g_pt.ev[c];
        if (cudaEventSynchronize(e[3]) != cudaSuccess) return -1;
        for (int k = 0; k < 3; k++) {
            float ms = 0;
            if (cudaEventElapsedTime(&ms, e[k], e[k + 1]) != cudaSuccess) return -1;
            ms_sums[k] += ms;
        }
    }
    *calls = g_pt.calls;
    return 0;
}

uint64_t partition_scratch_bytes(uint64_t n, uint32_t G, int out_width) {
    return layout(n, G, out_width).total;
}

static int env_int(const char* name, int dflt) {  // launch-shape knobs (tools/synth_perf.py)
    const char* e = std::getenv(name);
    return e && std::atoi(e) > 0 ? std::atoi(e) : dflt;
}

cudaError_t launch_query_partitioned(const DevIndex& ix0, int gamma_kind, bool pow2,
                                     const uint64_t* keys, int src_kind, uint64_t seq_words,
                                     uint32_t kbits, void* out, int out_width, uint64_t n,
                                     int minimal, uint32_t G, void* scratch, cudaStream_t s,
                                     int sms) {
    if (n == 0) return cudaSuccess;
    if (G < 1 || G > (uint32_t)kMaxGroups) return cudaErrorInvalidValue;
    // Pass B reads the pilots with evict_last: the L2 of each die then keeps its own copy of
    // the far die's lines of the current slice (measured at config 3: L2 fabric requests
    // 610M -> 101M, pass B 5.96 -> 4.84 ms); lines of earlier slices evict one another.
    DevIndex ix = ix0;
    ix.window_bytes = 0;
    ix.pilot_evict_normal = env_int("PH_GPU_PB_NORMAL", 0) ? 1 : 0;
    ix.cold_evict_first = 0;
    const Layout L = layout(n, G, out_width);
    uint8_t* base = static_cast<uint8_t*>(scratch);
    auto* ctrl = reinterpret_cast<unsigned long long*>(base);
    auto* runoff = reinterpret_cast<uint64_t*>(base + L.o_runoff);
    auto* runcnt = reinterpret_cast<uint16_t*>(base + L.o_runcnt);
    auto* bins = reinterpret_cast<uint64_t*>(base + L.o_bins);
    auto* bpos = reinterpret_cast<uint16_t*>(base + L.o_bpos);
    void* slots = base + L.o_slots;

    pt_record(0, s);
    cudaError_t e = cudaMemsetAsync(ctrl, 0, kCtrlWords * 8, s);
    if (e != cudaSuccess) return e;
#ifdef PH_CHECKS
    {
        const ChkBounds cb{L.nent, n, src_kind == 1 ? seq_words : n, L.ntiles};
        cudaMemcpyToSymbolAsync(g_chk_b, &cb, sizeof(cb), 0, cudaMemcpyHostToDevice, s);
        cudaMemsetAsync(base + L.total - kCanaryBytes, 0xA5, kCanaryBytes, s);
    }
#endif
    // A: bin the keys by group
    const size_t smem_a = kTileKeys * (8 + 4);
    // (per device and cheap: set on every call)
    cudaFuncSetAttribute(k_bin<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_a);
    cudaFuncSetAttribute(k_bin<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_a);
    const uint64_t want = L.ntiles;
    const int grid_a = (int)(want < (uint64_t)sms * kBinCtas ? want : (uint64_t)sms * kBinCtas);
    nvtx_mark("partitioned: pass A (bin)");
    const bool tma = G <= (uint32_t)kTmaGroups && !std::getenv("PH_GPU_NO_TMA") &&
                     (src_kind == 1 || (reinterpret_cast<uintptr_t>(keys) & 15) == 0);
    if (tma) {
        const uint64_t ctas =
            (uint64_t)sms * env_int("PH_GPU_PART_A_CTAS", src_kind == 1 ? PH_BIN_KMER_CTAS : 2);
        const int grid_t = (int)(want < ctas ? want : ctas);
        if (src_kind == 1) {
            constexpr size_t sm = bin_tma_smem<1>();
            cudaFuncSetAttribute(k_bin_tma<kBinTmaThreads, 1>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            k_bin_tma<kBinTmaThreads, 1><<<grid_t, kBinTmaThreads, sm, s>>>(
                keys, n, seq_words, kbits, ix.seed, G, L.cap, ctrl, runoff, runcnt, bins, bpos);
        } else {
            constexpr size_t sm = bin_tma_smem<0>();
            cudaFuncSetAttribute(k_bin_tma<kBinTmaThreads, 0>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            k_bin_tma<kBinTmaThreads, 0><<<grid_t, kBinTmaThreads, sm, s>>>(
                keys, n, 0, 0, ix.seed, G, L.cap, ctrl, runoff, runcnt, bins, bpos);
        }
    } else if (src_kind == 1) {
        k_bin<1><<<grid_a, kBinThreads, smem_a, s>>>(keys, n, seq_words, kbits, ix.seed, G, L.cap,
                                                   ctrl, runoff, runcnt, bins, bpos);
    } else {
        k_bin<0><<<grid_a, kBinThreads, smem_a, s>>>(keys, n, 0, 0, ix.seed, G, L.cap, ctrl, runoff,
                                                   runcnt, bins, bpos);
    }
    note_launch();
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    // B: the query arithmetic (and remap_slot) over the group regions, one L2-resident
    // pilot slice after another
    pt_record(1, s);
    nvtx_mark("partitioned: pass B (query regions)");
    const int b_per_sm = env_int("PH_GPU_PART_B_CTAS", 4);
    e = out_width == 4
            ? launch_regions(ix, gamma_kind, pow2, G, L.cap, L.nent, ctrl, bins,
                             static_cast<uint32_t*>(slots), minimal, s, sms, b_per_sm)
            : launch_regions(ix, gamma_kind, pow2, G, L.cap, L.nent, ctrl, bins,
                             static_cast<uint64_t*>(slots), minimal, s, sms, b_per_sm);
    if (e != cudaSuccess) return e;
    pt_record(2, s);
    // C: back to input order
    nvtx_mark("partitioned: pass C (unbin)");
    const size_t sm4 = UnbinTma<uint32_t>::kSmem, sm8 = UnbinTma<uint64_t>::kSmem;
    cudaFuncSetAttribute(k_unbin_tma<uint32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm4);
    cudaFuncSetAttribute(k_unbin_tma<uint64_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm8);
    const uint64_t ctas = (uint64_t)sms * (out_width == 4 ? env_int("PH_GPU_PART_C_CTAS", 3) : 1);
    const int grid_c = (int)(want < ctas ? want : ctas);
    if (out_width == 4)
        k_unbin_tma<uint32_t><<<grid_c, kBinThreads, sm4, s>>>(
            n, G, runoff, runcnt, bpos, static_cast<const uint32_t*>(slots), static_cast<uint32_t*>(out));
    else
        k_unbin_tma<uint64_t><<<grid_c, kBinThreads, sm8, s>>>(
            n, G, runoff, runcnt, bpos, static_cast<const uint64_t*>(slots), static_cast<uint64_t*>(out));
    note_launch();
    pt_record(3, s);
#ifdef PH_CHECKS
    k_canary_check<<<1, 256, 0, s>>>(reinterpret_cast<const uint32_t*>(base + L.total - kCanaryBytes),
                                     (uint32_t)(kCanaryBytes / 4));
#endif
    return cudaGetLastError();
}

// Violations counted by a checked build since the last call (and the source line of the
// first); -1 in normal builds.
int check_errors(uint64_t* count, uint64_t* line) {
#ifdef PH_CHECKS
    unsigned long long h[2] = {0, 0};
    if (cudaMemcpyFromSymbol(h, g_chk, sizeof(h)) != cudaSuccess) return -2;
    const unsigned long long z[2] = {0, 0};
    cudaMemcpyToSymbol(g_chk, z, sizeof(z));
    *count = h[0];
    *line = h[1];
    uint64_t sc = 0, sl = 0;  // the pilot-search kernel's counters (ph_search.cu)
    if (search_check_errors(&sc, &sl) == 0 && sc) {
        if (!*count) *line = 1000000 + sl;  // (lines of ph_search.cu are reported + 1e6)
        *count += sc;
    }
    return 0;
#else
    *count = *line = 0;
    return -1;
#endif
}

}  // namespace phg
