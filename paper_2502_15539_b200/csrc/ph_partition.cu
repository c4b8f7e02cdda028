// ph_partition.cu — the partitioned query path for DRAM-sized indexes.
//
// When the pilot array is far larger than what the L2 holds for random access (~64 MB),
// every direct query pays a DRAM row activation for its 1-byte pilot read (~57 G/s over
// 333 MB). This path turns those random DRAM reads into streaming passes plus L2-resident
// random reads. Keys are binned by hash group g = hi(G * h): group g's keys only use parts
// [gP/G, (g+1)P/G], a contiguous ~P*B/G-byte slice of the pilots that fits in the L2.
//
//   A  bin     per 4096-key tile: ranks by group in shared memory, one global atomicAdd
//              per (tile, group) to reserve a run in that group's region, then the runs are
//              written from shared memory with coalesced stores: entry = (key, position in
//              the tile as u16). Run (offset, length) -> runoff/runcnt[tile][g].
//   B  query   the ordinary query kernel (L2-resident tuning), one launch per group region
//              (so the warps of a launch only touch that group's pilot slice), then one
//              over the spill; answers into slots[] at the same entry index.
//   C  unbin   per tile: the G runs' (position, slot) pairs are scattered into a shared
//              memory tile, which is then written to out[] with coalesced stores.
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

#include <cmath>
#include <cstdint>

#include "ph_device.cuh"
#include "ph_kernels.h"

namespace phg {

constexpr int kBinThreads = 256;
constexpr int kBinPerThread = 16;
constexpr uint32_t kTileKeys = kBinThreads * kBinPerThread;  // 4096 keys per tile
constexpr int kBinCtas = 4;    // CTAs per SM (registers: 64 per thread)
constexpr int kUnbinCtas = 5;
constexpr int kMaxGroups = 64;
// ctrl[]: per-group cursors [0, kMaxGroups), spill cursor
constexpr int kCtrlSpill = kMaxGroups;
constexpr int kCtrlWords = kMaxGroups + 1;

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
    extern __shared__ __align__(16) uint8_t smem[];
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
                    uint64_t off = 0;
                    if (c) {
                        off = atomicAdd(ctrl + g, (unsigned long long)c);
                        off = off + c <= cap
                                  ? g * cap + off
                                  : G * cap + atomicAdd(ctrl + kCtrlSpill, (unsigned long long)c);
                    }
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

// Pass C. Per tile: the G runs are laid end to end (run g at lbase[g]); rid[e] names the
// run of staged entry e. Every thread issues its 16 (position, slot) loads before storing
// any into the shared-memory tile, which is then written out in order.
template <class OutT>
__global__ void __launch_bounds__(kBinThreads, sizeof(OutT) == 4 ? kUnbinCtas : kUnbinCtas - 1) k_unbin(
    uint64_t n, uint32_t G, const uint64_t* __restrict__ runoff,
    const uint16_t* __restrict__ runcnt, const uint16_t* __restrict__ bpos,
    const OutT* __restrict__ slots, OutT* __restrict__ out) {
    extern __shared__ __align__(16) uint8_t smem[];
    OutT* stage = reinterpret_cast<OutT*>(smem);
    uint8_t* rid = reinterpret_cast<uint8_t*>(stage + kTileKeys);
    __shared__ uint32_t rc[kMaxGroups];
    __shared__ uint32_t lbase[kMaxGroups];
    __shared__ uint64_t delta[kMaxGroups];  // run offset - staged offset
    const unsigned tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t ntiles = (n + kTileKeys - 1) / kTileKeys;
    for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const uint64_t t0 = t * kTileKeys;
        const uint32_t valid = (uint32_t)(n - t0 < kTileKeys ? n - t0 : kTileKeys);
        if (warp == 0) {
            const uint32_t g0 = 2 * lane;
            const uint32_t c0 = g0 < G ? __ldg(runcnt + t * G + g0) : 0;
            const uint32_t c1 = g0 + 1 < G ? __ldg(runcnt + t * G + g0 + 1) : 0;
            const uint64_t o0 = g0 < G ? __ldg(runoff + t * G + g0) : 0;
            const uint64_t o1 = g0 + 1 < G ? __ldg(runoff + t * G + g0 + 1) : 0;
            uint32_t x = c0 + c1;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(kFull, x, o);
                if (lane >= (unsigned)o) x += y;
            }
            x -= c0 + c1;
            lbase[g0] = x;
            lbase[g0 + 1] = x + c0;
            delta[g0] = o0 - x;
            delta[g0 + 1] = o1 - (x + c0);
            rc[g0] = c0;
            rc[g0 + 1] = c1;
        }
        __syncthreads();
        for (uint32_t g = warp; g < G; g += kBinThreads / 32) {
            const uint32_t c = rc[g], lb = lbase[g];
            for (uint32_t i = lane; i < c; i += 32) rid[lb + i] = (uint8_t)g;
        }
        __syncthreads();
        uint16_t pv[kBinPerThread];
        OutT sv[kBinPerThread];
#pragma unroll
        for (int j = 0; j < kBinPerThread; j++) {
            const uint32_t e = (uint32_t)j * kBinThreads + tid;
            if (e < valid) {
                const uint64_t src = delta[rid[e]] + e;
                pv[j] = __ldcs(bpos + src);
                sv[j] = __ldcs(slots + src);
            }
        }
#pragma unroll
        for (int j = 0; j < kBinPerThread; j++)
            if ((uint32_t)j * kBinThreads + tid < valid) stage[pv[j]] = sv[j];
        __syncthreads();
        {
#pragma unroll 4
            for (int j = 0; j < kBinPerThread; j++) {
                const uint32_t e = (uint32_t)j * kBinThreads + tid;
                if (e < valid) st_stream(out + t0 + e, stage[e]);
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
namespace {
struct Layout {
    uint64_t cap, ntiles, nent;
    uint64_t o_runoff, o_runcnt, o_bins, o_bpos, o_slots, total;
};
Layout layout(uint64_t n, uint32_t G, int out_width) {
    auto al = [](uint64_t b) { return (b + 255) & ~uint64_t{255}; };
    Layout L;
    const uint64_t per = (n + G - 1) / G;
    L.cap = per + 16 * (uint64_t)std::ceil(std::sqrt((double)per)) + kTileKeys;
    L.cap = (L.cap + 255) & ~uint64_t{255};
    L.ntiles = (n + kTileKeys - 1) / kTileKeys;
    L.nent = G * L.cap + n;
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
    L.total = o;
    return L;
}
}  // namespace

uint64_t partition_scratch_bytes(uint64_t n, uint32_t G, int out_width) {
    return layout(n, G, out_width).total;
}

cudaError_t launch_query_partitioned(const DevIndex& ix, int gamma_kind, bool pow2,
                                     const uint64_t* keys, int src_kind, uint64_t seq_words,
                                     uint32_t kbits, void* out, int out_width, uint64_t n,
                                     int minimal, uint32_t G, void* scratch, cudaStream_t s,
                                     int sms, const RemapList& rl) {
    if (n == 0) return cudaSuccess;
    if (G < 1 || G > (uint32_t)kMaxGroups) return cudaErrorInvalidValue;
    const Layout L = layout(n, G, out_width);
    uint8_t* base = static_cast<uint8_t*>(scratch);
    auto* ctrl = reinterpret_cast<unsigned long long*>(base);
    auto* runoff = reinterpret_cast<uint64_t*>(base + L.o_runoff);
    auto* runcnt = reinterpret_cast<uint16_t*>(base + L.o_runcnt);
    auto* bins = reinterpret_cast<uint64_t*>(base + L.o_bins);
    auto* bpos = reinterpret_cast<uint16_t*>(base + L.o_bpos);
    void* slots = base + L.o_slots;

    cudaError_t e = cudaMemsetAsync(ctrl, 0, kCtrlWords * 8, s);
    if (e != cudaSuccess) return e;
    const size_t smem_a = kTileKeys * (8 + 4);
    // (per device and cheap: set on every call)
    cudaFuncSetAttribute(k_bin<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_a);
    cudaFuncSetAttribute(k_bin<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_a);
    cudaFuncSetAttribute(k_unbin<uint64_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(kTileKeys * 9));
    const uint64_t want = L.ntiles;
    const int grid_a = (int)(want < (uint64_t)sms * kBinCtas ? want : (uint64_t)sms * kBinCtas);
    const uint64_t ctas_c = (uint64_t)sms * (out_width == 4 ? kUnbinCtas : kUnbinCtas - 1);
    const int grid_c = (int)(want < ctas_c ? want : ctas_c);
    if (src_kind == 1)
        k_bin<1><<<grid_a, kBinThreads, smem_a, s>>>(keys, n, seq_words, kbits, ix.seed, G, L.cap,
                                                   ctrl, runoff, runcnt, bins, bpos);
    else
        k_bin<0><<<grid_a, kBinThreads, smem_a, s>>>(keys, n, 0, 0, ix.seed, G, L.cap, ctrl, runoff,
                                                   runcnt, bins, bpos);
    note_launch();
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    // B: the query kernel over the entries, one L2-sized pilot slice after another
    // (no persisting window and evict_normal pilots: earlier slices must be evictable)
    DevIndex ixb = ix;
    ixb.window_bytes = 0;
    ixb.pilot_evict_normal = 1;
    ixb.cold_evict_first = 0;
    uint8_t* sl = static_cast<uint8_t*>(slots);
    for (uint32_t g = 0; g <= G; g++) {  // g == G: the spill region
        const uint64_t off = g * L.cap;
        e = launch_query_bins(ixb, gamma_kind, pow2, bins + off, ctrl + (g < G ? g : kCtrlSpill), g < G ? L.cap : n,
                              sl + off * out_width, out_width, minimal, s, sms, rl);
        if (e != cudaSuccess) return e;
    }
    const size_t smem_c = kTileKeys * (size_t)(out_width + 1);
    if (out_width == 4)
        k_unbin<uint32_t><<<grid_c, kBinThreads, smem_c, s>>>(n, G, runoff, runcnt, bpos,
                                                            static_cast<const uint32_t*>(slots),
                                                            static_cast<uint32_t*>(out));
    else
        k_unbin<uint64_t><<<grid_c, kBinThreads, smem_c, s>>>(n, G, runoff, runcnt, bpos,
                                                            static_cast<const uint64_t*>(slots),
                                                            static_cast<uint64_t*>(out));
    note_launch();
    return cudaGetLastError();
}

}  // namespace phg
