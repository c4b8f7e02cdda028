// ph_sort.cu — hand-written MSD radix sort of the u64 build hashes (construction assist,
// SURVEY §8f-3; off the query path).
//
// The reference sorts each part's hashes with std::sort after scatter_to_parts
// (engine.hpp:412-474, :505-513). part = hi(P*h) is monotone in h, so one ascending sort of
// all n hashes gives exactly that part-major, per-part-sorted array. The sort here:
//
//   level split  (k_msd_hist + k_msd_scatter)  per segment, the next 8 bits of h: a
//                histogram pass, an exclusive scan on the host, and a scatter pass that
//                ranks each 4096-key tile by digit in shared memory, reserves one run per
//                (tile, digit) with a global atomicAdd and writes every run contiguously
//                from a digit-ordered shared-memory stage. The first level hashes the keys
//                on the fly (h = C*(key^seed), hash.hpp:27), so there is no hash pass.
//   segment sort (k_seg_sort)  one 1024-thread CTA per segment of <= 24576 hashes that
//                share their top bits: rank by the next 12 bits in shared memory, place,
//                insertion-sort each of the 4096 bins (uniform hashes put ~4 keys in a
//                bin), write back.
//
// At n = 1e9 that is two levels (256 x 256 segments of ~15k keys) and one segment-sort
// pass: 8 (hist) + 16 (scatter) per level + 16 (segment sort) = 56 B of DRAM per key
// (the first hist pass reads keys, not hashes). Skewed inputs cannot break it, only slow
// it: a segment larger than the cap, or whose bins exceed 64 keys, is split by another
// 8 bits; after all 64 bits every remaining segment holds one value.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <vector>

#include "ph_device.cuh"
#include "ph_kernels.h"

namespace phg {
namespace {

constexpr int kSplitThreads = 512;
constexpr int kTile = 4096;                  // keys per scatter tile (8 per thread)
constexpr uint64_t kChunk = 16 * kTile;      // keys per split work item
constexpr int kSegThreads = 1024;
constexpr uint32_t kSegCap = 24576;          // keys per segment sort (24 per thread)
constexpr int kSegPer = kSegCap / kSegThreads;
constexpr int kSubBits = 12;                 // bins of the segment sort
constexpr uint32_t kSubBins = 1u << kSubBits;
constexpr uint32_t kMaxBin = 64;             // larger bins: split the segment instead
constexpr size_t kSegSmem = kSegCap * 8 + kSubBins * 4 + 64;

struct WorkItem {   // one CTA of a split pass: keys [start, start+len) of segment seg
    uint64_t start;
    uint32_t len;
    uint32_t seg;
};
struct SegItem {    // one CTA of the segment sort
    uint64_t start;
    uint32_t len;
    uint32_t id;
};

template <bool HASH, bool NC = true>
__device__ __forceinline__ uint64_t load_h(const uint64_t* src, uint64_t i, uint64_t seed) {
    const uint64_t v = NC ? __ldg(src + i) : src[i];
    return HASH ? kC * (v ^ seed) : v;  // hash_int, hash.hpp:27
}

// Exclusive scan of n (multiple of 32, <= 32 * warps) shared counters into out, by the
// first n threads; returns nothing. All threads must call (two barriers).
__device__ __forceinline__ void block_exscan(const uint32_t* cnt, uint32_t* out, int n,
                                             uint32_t* wsum) {
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    uint32_t v = t < n ? cnt[t] : 0, inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += u;
    }
    if (t < n && lane == 31) wsum[w] = inc;
    __syncthreads();
    if (t < n) {
        uint32_t base = 0;
        for (int i = 0; i < w; i++) base += wsum[i];
        out[t] = base + inc - v;
    }
    __syncthreads();
}

template <bool HASH>
__global__ void __launch_bounds__(kSplitThreads) k_msd_hist(const uint64_t* __restrict__ src,
                                                            const WorkItem* __restrict__ items,
                                                            int shift, uint64_t seed,
                                                            unsigned long long* __restrict__ hist) {
    __shared__ uint32_t cnt[256];
    if (threadIdx.x < 256) cnt[threadIdx.x] = 0;
    __syncthreads();
    const WorkItem w = items[blockIdx.x];
    for (uint32_t i = threadIdx.x; i < w.len; i += kSplitThreads)
        atomicAdd(&cnt[(load_h<HASH>(src, w.start + i, seed) >> shift) & 255], 1u);
    __syncthreads();
    if (threadIdx.x < 256 && cnt[threadIdx.x])
        atomicAdd(hist + (uint64_t)w.seg * 256 + threadIdx.x, (unsigned long long)cnt[threadIdx.x]);
}

template <bool HASH>
__global__ void __launch_bounds__(kSplitThreads) k_msd_scatter(
    const uint64_t* __restrict__ src, uint64_t* __restrict__ dst,
    const WorkItem* __restrict__ items, int shift, uint64_t seed,
    unsigned long long* __restrict__ cursor) {
    __shared__ uint64_t stage[kTile];
    __shared__ uint32_t cnt[256], pre[256], wsum[16];
    __shared__ unsigned long long base[256];
    const WorkItem w = items[blockIdx.x];
    const int t = threadIdx.x;
    for (uint32_t t0 = 0; t0 < w.len; t0 += kTile) {
        const uint32_t m = min((uint32_t)kTile, w.len - t0);
        if (t < 256) cnt[t] = 0;
        __syncthreads();
        uint64_t h[kTile / kSplitThreads];
        uint32_t rk[kTile / kSplitThreads];
#pragma unroll
        for (int r = 0; r < kTile / kSplitThreads; r++) {
            const uint32_t i = r * kSplitThreads + t;
            if (i < m) {
                h[r] = load_h<HASH>(src, w.start + t0 + i, seed);
                rk[r] = atomicAdd(&cnt[(h[r] >> shift) & 255], 1u);
            }
        }
        __syncthreads();
        if (t < 256)  // this tile's run of digit t in the destination
            base[t] = cnt[t] ? atomicAdd(cursor + (uint64_t)w.seg * 256 + t,
                                         (unsigned long long)cnt[t]) : 0;
        block_exscan(cnt, pre, 256, wsum);
#pragma unroll
        for (int r = 0; r < kTile / kSplitThreads; r++) {
            const uint32_t i = r * kSplitThreads + t;
            if (i < m) stage[pre[(h[r] >> shift) & 255] + rk[r]] = h[r];
        }
        __syncthreads();
        for (uint32_t j = t; j < m; j += kSplitThreads) {  // runs leave contiguously
            const uint64_t v = stage[j];
            const uint32_t d = (v >> shift) & 255;
            dst[base[d] + (j - pre[d])] = v;
        }
        __syncthreads();
    }
}

// Sorts each segment (all its hashes share the bits above `shift`) into dst at the same
// positions. Bins are the next 12 bits below `shift` (all of them when shift <= 12, and then
// every bin holds one value). A segment with a bin over kMaxBin keys is left for another
// split level: its id goes to redo[].
template <bool HASH>
__global__ void __launch_bounds__(kSegThreads, 1) k_seg_sort(
    const uint64_t* src, uint64_t* dst,  // may alias (in place)
    const SegItem* __restrict__ segs, int shift, uint64_t seed, uint32_t* __restrict__ redo,
    uint32_t* __restrict__ redo_n) {
    extern __shared__ __align__(16) uint8_t smem[];
    uint64_t* buf = reinterpret_cast<uint64_t*>(smem);
    uint32_t* cnt = reinterpret_cast<uint32_t*>(smem + kSegCap * 8);
    __shared__ uint32_t wsum[32], maxbin;
    const SegItem s = segs[blockIdx.x];
    const int t = threadIdx.x;
    const int bshift = shift > kSubBits ? shift - kSubBits : 0;
    const uint64_t bmask = shift >= kSubBits ? (kSubBins - 1) : ((1ull << shift) - 1);
#pragma unroll
    for (int b = t; b < (int)kSubBins; b += kSegThreads) cnt[b] = 0;
    if (t == 0) maxbin = 0;
    __syncthreads();
    uint32_t rk[kSegPer / 2];  // two 16-bit ranks per word (ranks < kSegCap < 2^16)
#pragma unroll
    for (int r = 0; r < kSegPer; r++) {
        const uint32_t i = r * kSegThreads + t;
        uint32_t q = 0;
        if (i < s.len) q = atomicAdd(&cnt[(load_h<HASH, false>(src, s.start + i, seed) >> bshift) & bmask], 1u);
        if (r & 1) rk[r >> 1] |= q << 16; else rk[r >> 1] = q;
    }
    __syncthreads();
    // exclusive scan of the 4096 bins: 4 consecutive bins per thread
    uint32_t c4[4], sum = 0, mx = 0;
#pragma unroll
    for (int k = 0; k < 4; k++) {
        c4[k] = cnt[t * 4 + k];
        sum += c4[k];
        mx = max(mx, c4[k]);
    }
    {
        const int lane = t & 31, w = t >> 5;
        uint32_t inc = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += u;
        }
        if (lane == 31) wsum[w] = inc;
        if (shift > kSubBits && mx > kMaxBin) atomicMax(&maxbin, mx);
        __syncthreads();
        uint32_t base = 0;
        for (int i = 0; i < w; i++) base += wsum[i];
        base += inc - sum;
#pragma unroll
        for (int k = 0; k < 4; k++) {
            cnt[t * 4 + k] = base;  // now the bin's first position
            base += c4[k];
        }
    }
    __syncthreads();
    if (maxbin) {  // skewed segment: split it further instead
        if (t == 0) redo[atomicAdd(redo_n, 1u)] = s.id;
        return;
    }
#pragma unroll
    for (int r = 0; r < kSegPer; r++) {
        const uint32_t i = r * kSegThreads + t;
        if (i < s.len) {  // second read of the segment: an L2 hit
            const uint64_t h = load_h<HASH, false>(src, s.start + i, seed);
            const uint32_t q = (rk[r >> 1] >> ((r & 1) * 16)) & 0xffffu;
            buf[cnt[(h >> bshift) & bmask] + q] = h;
        }
    }
    __syncthreads();
    if (shift > kSubBits) {  // insertion sort of bins 4t .. 4t+3 (each <= kMaxBin keys)
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const uint32_t lo = cnt[t * 4 + k];
            const uint32_t hi = t * 4 + k + 1 < (int)kSubBins ? cnt[t * 4 + k + 1] : s.len;
            for (uint32_t i = lo + 1; i < hi; i++) {
                const uint64_t v = buf[i];
                uint32_t j = i;
                while (j > lo && buf[j - 1] > v) {
                    buf[j] = buf[j - 1];
                    j--;
                }
                buf[j] = v;
            }
        }
        __syncthreads();
    }
    for (uint32_t j = t; j < s.len; j += kSegThreads) dst[s.start + j] = buf[j];
}

struct Seg {
    uint64_t start, len;
};

template <class T>
cudaError_t upload(const std::vector<T>& v, T** d, cudaMemPool_t pool, cudaStream_t s) {
    cudaError_t e = cudaMallocFromPoolAsync(reinterpret_cast<void**>(d), std::max<size_t>(1, v.size()) * sizeof(T), pool, s);
    if (e == cudaSuccess && !v.empty())
        e = cudaMemcpyAsync(*d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s);
    return e;
}

}  // namespace

// Sorts h = C*(keys[i]^seed) for i < n ascending into out (n*8 bytes); tmp is n*8 bytes of
// scratch. Synchronous on s (the split levels need their histograms on the host).
cudaError_t sort_hashes_u64(const uint64_t* keys, uint64_t n, uint64_t seed, uint64_t* out,
                            uint64_t* tmp, cudaMemPool_t pool, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(k_seg_sort<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSegSmem);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_seg_sort<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSegSmem);
    if (e != cudaSuccess) return e;
    // depth 0 reads the keys (hashing them); depth d >= 1 lives in tmp (odd) or out (even)
    auto where = [&](int depth) -> const uint64_t* { return depth == 0 ? keys : (depth & 1) ? tmp : out; };
    std::vector<Seg> level{{0, n}};
    int shift = 64;
    for (int depth = 0; !level.empty(); depth++, shift -= 8) {
        const uint64_t* src = where(depth);
        std::vector<Seg> split;
        std::vector<SegItem> small;
        for (const Seg& g : level) {
            if (g.len == 0) continue;
            if (g.len <= kSegCap) small.push_back({g.start, (uint32_t)g.len, (uint32_t)small.size()});
            else if (shift == 0) {  // 64 bits consumed: one repeated value
                if (src != out)
                    e = cudaMemcpyAsync(out + g.start, src + g.start, g.len * 8, cudaMemcpyDeviceToDevice, s);
            } else {
                split.push_back(g);
            }
        }
        if (e != cudaSuccess) return e;
        if (!small.empty()) {  // segment sort; skewed segments come back through redo
            SegItem* d_items = nullptr;
            uint32_t* d_redo = nullptr;
            e = upload(small, &d_items, pool, s);
            if (e == cudaSuccess) e = cudaMallocFromPoolAsync(reinterpret_cast<void**>(&d_redo), (small.size() + 1) * 4, pool, s);
            if (e == cudaSuccess) e = cudaMemsetAsync(d_redo, 0, 4, s);
            if (e == cudaSuccess) {
                if (depth == 0)
                    k_seg_sort<true><<<(unsigned)small.size(), kSegThreads, kSegSmem, s>>>(
                        src, out, d_items, shift, seed, d_redo + 1, d_redo);
                else
                    k_seg_sort<false><<<(unsigned)small.size(), kSegThreads, kSegSmem, s>>>(
                        src, out, d_items, shift, seed, d_redo + 1, d_redo);
                note_launch();
                e = cudaGetLastError();
            }
            uint32_t nredo = 0;
            if (e == cudaSuccess) e = cudaMemcpyAsync(&nredo, d_redo, 4, cudaMemcpyDeviceToHost, s);
            if (e == cudaSuccess) e = cudaStreamSynchronize(s);
            if (e == cudaSuccess && nredo) {
                std::vector<uint32_t> ids(nredo);
                e = cudaMemcpy(ids.data(), d_redo + 1, nredo * 4, cudaMemcpyDeviceToHost);
                for (uint32_t id : ids) split.push_back({small[id].start, small[id].len});
            }
            cudaFreeAsync(d_items, s);
            cudaFreeAsync(d_redo, s);
            if (e != cudaSuccess) return e;
        }
        if (split.empty()) break;
        // one split level over `split`: histogram, host scan, scatter into the other buffer
        std::vector<WorkItem> items;
        for (uint32_t g = 0; g < split.size(); g++)
            for (uint64_t c = 0; c < split[g].len; c += kChunk)
                items.push_back({split[g].start + c, (uint32_t)std::min(kChunk, split[g].len - c), g});
        WorkItem* d_items = nullptr;
        unsigned long long* d_hist = nullptr;
        const size_t nh = split.size() * 256;
        e = upload(items, &d_items, pool, s);
        if (e == cudaSuccess) e = cudaMallocFromPoolAsync(reinterpret_cast<void**>(&d_hist), nh * 8, pool, s);
        if (e == cudaSuccess) e = cudaMemsetAsync(d_hist, 0, nh * 8, s);
        const int dshift = shift - 8;
        if (e == cudaSuccess) {
            if (depth == 0)
                k_msd_hist<true><<<(unsigned)items.size(), kSplitThreads, 0, s>>>(src, d_items, dshift, seed, d_hist);
            else
                k_msd_hist<false><<<(unsigned)items.size(), kSplitThreads, 0, s>>>(src, d_items, dshift, seed, d_hist);
            note_launch();
            e = cudaGetLastError();
        }
        std::vector<unsigned long long> hist(nh);
        if (e == cudaSuccess) e = cudaMemcpyAsync(hist.data(), d_hist, nh * 8, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        std::vector<Seg> next;
        if (e == cudaSuccess) {
            for (size_t g = 0; g < split.size(); g++) {
                uint64_t at = split[g].start;
                for (int d = 0; d < 256; d++) {
                    const uint64_t c = hist[g * 256 + d];
                    hist[g * 256 + d] = at;  // cursor
                    if (c) next.push_back({at, c});
                    at += c;
                }
            }
            e = cudaMemcpyAsync(d_hist, hist.data(), nh * 8, cudaMemcpyHostToDevice, s);
        }
        uint64_t* dst = const_cast<uint64_t*>(where(depth + 1));
        if (e == cudaSuccess) {
            if (depth == 0)
                k_msd_scatter<true><<<(unsigned)items.size(), kSplitThreads, 0, s>>>(src, dst, d_items, dshift, seed, d_hist);
            else
                k_msd_scatter<false><<<(unsigned)items.size(), kSplitThreads, 0, s>>>(src, dst, d_items, dshift, seed, d_hist);
            note_launch();
            e = cudaGetLastError();
        }
        cudaFreeAsync(d_items, s);
        cudaFreeAsync(d_hist, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);  // hist (host vector) in flight
        if (e != cudaSuccess) return e;
        level.swap(next);
    }
    return cudaSuccess;
}

}  // namespace phg
