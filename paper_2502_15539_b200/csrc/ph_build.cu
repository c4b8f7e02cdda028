// ph_build.cu — device assist for the construction phases that precede the pilot search
// (SURVEY §8f-3). Not part of the query path; the pilot search stays on the CPU.
//
// For u64 keys one build attempt of the reference (construction.cpp:28-60, run_attempt)
// starts with three data-parallel phases:
//   hash_all          construction.cpp:98-111   H64{C * (key ^ seed)} (hash.hpp:27)
//   scatter_to_parts  engine.hpp:412-474        part = mul_hi(P, h); part-major order;
//                                               kOversubscribed if a part has > S keys
//   per-part sort     engine.hpp:505-518        std::sort of each part's slice, then
//                                               kDuplicateHashes on equal neighbours
// part = hi(P * h) is monotone in h, so sorting all hashes by h gives exactly the
// part-major arrangement with every part sorted. This file produces that array and the
// part offsets on the device: the hand-written MSD radix sort of ph_sort.cu (which hashes
// the keys in its first pass), and a kernel that writes the part boundaries and checks both
// failure conditions.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <mutex>

#include "ph_device.cuh"
#include "ph_kernels.h"

namespace phg {
namespace {

__global__ void __launch_bounds__(256) k_hash_u64(const uint64_t* __restrict__ keys, uint64_t n,
                                                  uint64_t seed, uint64_t* __restrict__ h) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        h[i] = kC * (keys[i] ^ seed);  // hash_int, hash.hpp:27
}

__device__ __forceinline__ uint64_t part_of(uint64_t P, uint64_t h) { return __umul64hi(P, h); }

// offsets[p] = first index of part p in the sorted hashes (offsets[P] = n): index i writes
// the offsets of the parts in (part(i-1), part(i)], so every offset is written once.
// Also flags equal neighbours (engine.hpp:507-513).
__global__ void __launch_bounds__(256) k_part_bounds(const uint64_t* __restrict__ h, uint64_t n,
                                                     uint64_t P, uint64_t* __restrict__ offsets,
                                                     int* __restrict__ status) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i <= n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t pi = i < n ? part_of(P, h[i]) : P;
        const uint64_t pprev = i > 0 ? part_of(P, h[i - 1]) + 1 : 0;
        for (uint64_t p = pprev; p <= pi && p <= P; p++) offsets[p] = i;
        if (i > 0 && i < n && h[i] == h[i - 1]) atomicOr(status, 2);
    }
}

// kOversubscribed (engine.hpp:437-443): a part holds more than S keys.
__global__ void __launch_bounds__(256) k_part_sizes(const uint64_t* __restrict__ offsets, uint64_t P,
                                                    uint64_t S, int* __restrict__ status) {
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < P;
         p += (uint64_t)gridDim.x * blockDim.x)
        if (offsets[p + 1] - offsets[p] > S) atomicOr(status, 1);
}

}  // namespace

// Scratch comes from a per-device pool that keeps its memory between calls (the sort
// needs ~n*8 bytes of it; remapping that on every call would cost more than the sort).
static cudaError_t scratch_pool(cudaMemPool_t* pool) {
    static cudaMemPool_t pools[64] = {};
    static std::mutex mu;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess || dev < 0 || dev >= 64) return e != cudaSuccess ? e : cudaErrorInvalidDevice;
    std::lock_guard<std::mutex> lock(mu);
    if (!pools[dev]) {
        cudaMemPoolProps props = {};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        if ((e = cudaMemPoolCreate(&pools[dev], &props)) != cudaSuccess) return e;
        uint64_t keep = UINT64_MAX;
        cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &keep);
    }
    *pool = pools[dev];
    return cudaSuccess;
}

cudaError_t sort_hashes_u64(const uint64_t* keys, uint64_t n, uint64_t seed, uint64_t* out,
                            uint64_t* tmp, cudaMemPool_t pool, cudaStream_t s);

cudaError_t build_prepare_u64(const uint64_t* keys, uint64_t n, uint64_t P, uint64_t S,
                              uint64_t seed, uint64_t* hashes, uint64_t* offsets, int* status,
                              cudaStream_t s, int sms) {
    *status = 0;
    int* d_status = nullptr;
    uint64_t* tmp = nullptr;
    cudaMemPool_t pool = nullptr;
    cudaError_t e = scratch_pool(&pool);
    if (e == cudaSuccess) e = cudaMallocFromPoolAsync(&d_status, sizeof(int), pool, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(d_status, 0, sizeof(int), s);
    if (e == cudaSuccess && n) e = cudaMallocFromPoolAsync(&tmp, n * 8, pool, s);
    const int grid = sms * 8;
    // hashes = sorted C*(key^seed) (all 64 bits: the part is the high-order function of h)
    if (e == cudaSuccess && n) e = sort_hashes_u64(keys, n, seed, hashes, tmp, pool, s);
    if (e == cudaSuccess) {
        k_part_bounds<<<grid, 256, 0, s>>>(hashes, n, P, offsets, d_status);
        note_launch();
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) {
        k_part_sizes<<<grid, 256, 0, s>>>(offsets, P, S, d_status);
        note_launch();
        e = cudaGetLastError();
    }
    int h_status = 0;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&h_status, d_status, sizeof(int), cudaMemcpyDeviceToHost, s);
    if (tmp) cudaFreeAsync(tmp, s);
    if (d_status) cudaFreeAsync(d_status, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    // as run_attempt (construction.cpp:42-52): an oversubscribed part fails the scatter
    // before any part is sorted
    *status = (h_status & 1) ? 1 : (h_status & 2) ? 2 : 0;
    return e;
}

// ---------------------------------------------------------------------------------------
// Bucket-size statistics (stats.cpp:59-61, recorded by group_buckets, engine.hpp:304-322):
// hist[s] = number of the P*B buckets that hold s of the keys.
// ---------------------------------------------------------------------------------------
namespace {

template <int G>
__global__ void __launch_bounds__(256) k_bucket_count(const DevIndex ix,
                                                      const uint64_t* __restrict__ keys,
                                                      uint64_t n, uint32_t* __restrict__ cnt) {
    const uint32_t P32 = (uint32_t)ix.P, B32 = (uint32_t)ix.B;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t h = kC * (keys[i] ^ ix.seed);  // hash_int, hash.hpp:27
        uint64_t x;
        const uint32_t part = (uint32_t)mul32x64(P32, h, x);  // part_and_bucket, bucket_fn.hpp:66-72
        const uint32_t bucket = bucket_of<G>(x, B32, ix.opt_table);
        atomicAdd(cnt + (uint64_t)part * B32 + bucket, 1u);
    }
}

constexpr int kHistBins = 64;  // per-block shared bins for sizes < 63
constexpr uint32_t kMaxHistSize = 1u << 24;

__global__ void __launch_bounds__(256) k_bucket_hist(const uint32_t* __restrict__ cnt,
                                                     uint64_t nb, unsigned long long* __restrict__ hist,
                                                     uint32_t* __restrict__ max_size) {
    __shared__ unsigned long long sh[kHistBins];
    if (threadIdx.x < kHistBins) sh[threadIdx.x] = 0;
    __syncthreads();
    uint32_t mx = 0;
    for (uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b < nb;
         b += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t c = cnt[b];
        mx = max(mx, c);
        if (c < kHistBins - 1) atomicAdd(&sh[c], 1ull);
        else atomicAdd(hist + min(c, kMaxHistSize), 1ull);  // rare large buckets
    }
    __syncthreads();
    if (threadIdx.x < kHistBins - 1 && sh[threadIdx.x]) atomicAdd(hist + threadIdx.x, sh[threadIdx.x]);
    atomicMax(max_size, mx);
}

template <int G>
cudaError_t bucket_count(const DevIndex& ix, const uint64_t* keys, uint64_t n, uint32_t* cnt,
                         cudaStream_t s, int sms) {
    k_bucket_count<G><<<sms * 8, 256, 0, s>>>(ix, keys, n, cnt);
    note_launch();
    return cudaGetLastError();
}

}  // namespace

cudaError_t bucket_size_hist(const DevIndex& ix, int gamma_kind, const uint64_t* keys, uint64_t n,
                             uint64_t* hist_out, uint64_t cap, uint64_t* len_out, cudaStream_t s,
                             int sms) {
    const uint64_t nb = ix.P * ix.B;
    cudaMemPool_t pool = nullptr;
    cudaError_t e = scratch_pool(&pool);
    uint32_t* cnt = nullptr;
    unsigned long long* hist = nullptr;  // counts for sizes 0..n (a bucket holds at most n keys)
    uint32_t* mx = nullptr;
    // sizes up to 2^24 (a bucket holds at most n keys); larger ones are reported as an error
    const uint64_t hbins = std::max<uint64_t>(std::min<uint64_t>(n, kMaxHistSize) + 1, kHistBins);
    if (e == cudaSuccess) e = cudaMallocFromPoolAsync(&cnt, nb * 4, pool, s);
    if (e == cudaSuccess) e = cudaMallocFromPoolAsync(&hist, hbins * 8 + 8, pool, s);
    if (e == cudaSuccess) {
        mx = reinterpret_cast<uint32_t*>(hist + hbins);
        e = cudaMemsetAsync(cnt, 0, nb * 4, s);
    }
    if (e == cudaSuccess) e = cudaMemsetAsync(hist, 0, hbins * 8 + 8, s);
    if (e == cudaSuccess && n) {
        switch (gamma_kind) {
            case 0: e = bucket_count<0>(ix, keys, n, cnt, s, sms); break;
            case 1: e = bucket_count<1>(ix, keys, n, cnt, s, sms); break;
            case 2: e = bucket_count<2>(ix, keys, n, cnt, s, sms); break;
            case 3: e = bucket_count<3>(ix, keys, n, cnt, s, sms); break;
            case 4: e = bucket_count<4>(ix, keys, n, cnt, s, sms); break;
            default: e = cudaErrorInvalidValue;
        }
    }
    if (e == cudaSuccess) {
        k_bucket_hist<<<sms * 8, 256, 0, s>>>(cnt, nb, hist, mx);
        note_launch();
        e = cudaGetLastError();
    }
    uint32_t h_mx = 0;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&h_mx, mx, 4, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e == cudaSuccess && h_mx > kMaxHistSize) e = cudaErrorNotSupported;
    if (e == cudaSuccess) {
        *len_out = (uint64_t)h_mx + 1;
        e = cudaMemcpy(hist_out, hist, std::min<uint64_t>(cap, *len_out) * 8, cudaMemcpyDeviceToHost);
    }
    if (hist) cudaFreeAsync(hist, s);
    if (cnt) cudaFreeAsync(cnt, s);
    return e;
}

}  // namespace phg
