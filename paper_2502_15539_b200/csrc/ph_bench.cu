// ph_bench.cu — measurement tools for bench.py and the GPU tests (NOT the product).
//
//  * synthetic query streams generated on the device (the workloads of
//    SURVEY §8d): corpus_u64 keys (reference corpus.hpp:14-16) in a seeded
//    Feistel-permuted order, or sampled with replacement;
//  * the random-sector gather microbenchmark that defines R_gather(F), the
//    pilot-gather roofline, using the same load instruction
//    and cache policy as the query kernel;
//  * a bijection checker (bitset + atomicOr old-bit detection).
#include <cuda_runtime.h>

#include <cstdint>

namespace {

constexpr uint64_t kGolden = 0x9e3779b97f4a7c15ULL;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t corpus_u64(uint64_t i, uint64_t gen_seed) {
    return mix64(gen_seed + (i + 1) * kGolden);
}
// Same function as oracle/ph_oracle.c pho_feistel_perm.
__host__ __device__ __forceinline__ uint64_t feistel(uint64_t i, uint64_t n, uint64_t seed,
                                                     unsigned h) {
    const uint64_t mask = (1ULL << h) - 1;
    uint64_t x = i;
    do {
        uint64_t L = x >> h, R = x & mask;
#pragma unroll
        for (uint64_t r = 0; r < 4; r++) {
            const uint64_t t = L ^ (mix64(R ^ (seed + (r + 1) * kGolden)) & mask);
            L = R;
            R = t;
        }
        x = (L << h) | R;
    } while (x >= n);
    return x;
}
unsigned feistel_half_bits(uint64_t n) {
    unsigned bits = 2;
    while (bits < 64 && (1ULL << bits) < n) bits += 2;
    return bits / 2;
}

__global__ void k_gen_perm(uint64_t* out, uint64_t start, uint64_t count, uint64_t n,
                           uint64_t gen_seed, uint64_t perm_seed, unsigned h) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
         i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = corpus_u64(feistel(start + i, n, perm_seed, h), gen_seed);
}
__global__ void k_gen_sample(uint64_t* out, uint64_t start, uint64_t count, uint64_t n,
                             uint64_t gen_seed, uint64_t sample_seed) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
         i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = corpus_u64(mix64(sample_seed + (start + i + 1) * kGolden) % n, gen_seed);
}
__global__ void k_gen_corpus(uint64_t* out, uint64_t start, uint64_t count, uint64_t gen_seed) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
         i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = corpus_u64(start + i, gen_seed);
}

// Uniform random 1-byte loads over [0, F): KPT independent loads per thread in
// flight, the query kernel's ld.global.nc + L2::evict_last policy.
template <int KPT>
__global__ void __launch_bounds__(256) k_gather(const uint8_t* __restrict__ buf, uint64_t F,
                                                uint64_t nloads, uint64_t seed, uint32_t* sink) {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * KPT;
    uint32_t acc = 0;
    for (uint64_t base = tid * KPT; base < nloads; base += stride) {
        uint32_t v[KPT];
#pragma unroll
        for (int j = 0; j < KPT; j++) {
            const uint64_t r = mix64(seed + (base + j) * kGolden);
            const uint64_t a = __umul64hi(r, F);
            uint16_t x = 0;
            if (base + j < nloads)
                asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u8 %0, [%1], %2;"
                             : "=h"(x) : "l"(buf + a), "l"(pol));
            v[j] = x;
        }
#pragma unroll
        for (int j = 0; j < KPT; j++) acc += v[j];
    }
    if (acc == 0x7fffffffu) *sink = acc;  // keep the loads alive
}

// Skewed gather: a fraction p_hot (out of 2^32) of the loads go uniformly to [0, F_hot),
// the rest uniformly to [F_hot, F). policy_mode: 0 = all evict_last, 1 = hot evict_last /
// cold evict_first, 2 = all normal (no hint).
__global__ void __launch_bounds__(256) k_gather_skew(const uint8_t* __restrict__ buf,
                                                     uint64_t F_hot, uint64_t F, uint32_t p_hot,
                                                     uint64_t nloads, uint64_t seed, int mode,
                                                     uint32_t* sink, const uint64_t* sin,
                                                     uint32_t* sout) {
    uint64_t pk, pc;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pk));
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pc));
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * 8;
    uint32_t acc = 0;
    for (uint64_t base = tid * 8; base < nloads; base += stride) {
        uint32_t v[8];
#pragma unroll
        for (int j = 0; j < 8; j++) {
            const uint64_t r = mix64(seed + (base + j) * kGolden);
            const bool hot = (uint32_t)r < p_hot;
            const uint64_t a = hot ? __umul64hi(r, F_hot) : F_hot + __umul64hi(r, F - F_hot);
            uint16_t x = 0;
            if (mode == 2) {
                asm volatile("ld.global.nc.L1::no_allocate.u8 %0, [%1];" : "=h"(x) : "l"(buf + a));
            } else {
                const uint64_t pol = (mode == 1 && !hot) ? pc : pk;
                asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u8 %0, [%1], %2;"
                             : "=h"(x) : "l"(buf + a), "l"(pol));
            }
            v[j] = x;
        }
        if (sin) {  // the query kernel's stream: 8 B in (evict_first) + 4 B out (.cs) per load
#pragma unroll
            for (int j = 0; j < 8; j++) {
                uint64_t kv;
                asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u64 %0, [%1], %2;"
                             : "=l"(kv) : "l"(sin + base + j), "l"(pc));
                asm volatile("st.global.cs.u32 [%0], %1;" ::"l"(sout + base + j), "r"((uint32_t)kv + v[j]));
            }
        }
#pragma unroll
        for (int j = 0; j < 8; j++) acc += v[j];
    }
    if (acc == 0x7fffffffu) *sink = acc;
}

// L1->XBAR port model (pass B's bound): per gather (uniform random 1-byte
// load over [0, F), evict_last), IN coalesced 8-byte words streamed in (evict_first) and one
// OUT-byte coalesced store (.cs; OUT = 0, 4 or 8). Measures how the L2-resident gather rate
// falls as streamed sectors share the SM's request port with the gathers.
template <int IN, int OUT>
__global__ void __launch_bounds__(256, 4) k_port(const uint8_t* __restrict__ buf, uint64_t F,
                                                 uint64_t nloads, uint64_t seed,
                                                 const uint64_t* __restrict__ sin, void* sout,
                                                 uint32_t* sink) {
    uint64_t pk, pc;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pk));
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pc));
    const unsigned lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    uint32_t acc = 0;
    for (uint64_t base = warp * 256; base + 256 <= nloads; base += nwarps * 256) {
        uint64_t kv[8];
        uint32_t v[8];
#pragma unroll
        for (int j = 0; j < 8; j++) {
            kv[j] = 0;
#pragma unroll
            for (int w = 0; w < IN; w++) {
                uint64_t t;
                asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u64 %0, [%1], %2;"
                             : "=l"(t) : "l"(sin + (base + j * 32 + lane) * IN + w), "l"(pc));
                kv[j] ^= t;
            }
        }
#pragma unroll
        for (int j = 0; j < 8; j++) {
            const uint64_t r = mix64(seed + (base + j * 32 + lane) * kGolden + (IN ? (kv[j] & 1) : 0));
            uint16_t x;
            asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u8 %0, [%1], %2;"
                         : "=h"(x) : "l"(buf + __umul64hi(r, F)), "l"(pk));
            v[j] = x;
        }
#pragma unroll
        for (int j = 0; j < 8; j++) {
            if (OUT == 4)
                asm volatile("st.global.cs.u32 [%0], %1;" ::"l"((uint32_t*)sout + base + j * 32 + lane),
                             "r"(v[j] + (uint32_t)kv[j]) : "memory");
            else if (OUT == 42) {  // 4 B per gather, two per store (pass B's st.global.cs.v2.u32)
                if (j & 1)
                    asm volatile("st.global.cs.v2.u32 [%0], {%1,%2};" ::"l"((uint32_t*)sout + base + (j >> 1) * 64 + lane * 2),
                                 "r"(v[j - 1] + (uint32_t)kv[j - 1]), "r"(v[j] + (uint32_t)kv[j]) : "memory");
            } else if (OUT == 44) {  // 4 B per gather, four per store
                if ((j & 3) == 3)
                    asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"((uint32_t*)sout + base + (j >> 2) * 128 + lane * 4),
                                 "r"(v[j - 3] + (uint32_t)kv[j - 3]), "r"(v[j - 2] + (uint32_t)kv[j - 2]),
                                 "r"(v[j - 1] + (uint32_t)kv[j - 1]), "r"(v[j] + (uint32_t)kv[j]) : "memory");
            }
            else if (OUT == 8)
                asm volatile("st.global.cs.u64 [%0], %1;" ::"l"((uint64_t*)sout + base + j * 32 + lane),
                             "l"(kv[j] + v[j]) : "memory");
            else
                acc += v[j] + (uint32_t)kv[j];
        }
    }
    if (acc == 0x7fffffffu) *sink = acc;
}

// The same as k_port<1, 4>, but each warp stages its 256 four-byte outputs in shared memory
// and lane 0 sends them with one 1 KiB bulk store (cp.async.bulk.global.shared::cta), double
// buffered: does the TMA store path load the SM's request port less than per-thread stores?
__global__ void __launch_bounds__(256, 4) k_port_bulk(const uint8_t* __restrict__ buf, uint64_t F,
                                                      uint64_t nloads, uint64_t seed,
                                                      const uint64_t* __restrict__ sin,
                                                      uint32_t* __restrict__ sout, uint32_t* sink) {
    __shared__ __align__(128) uint32_t stage[8][2][256];
    uint64_t pk, pc;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pk));
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pc));
    const unsigned lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    uint32_t it = 0;
    for (uint64_t base = warp * 256; base + 256 <= nloads; base += nwarps * 256, it++) {
        uint64_t kv[8];
        uint32_t v[8];
#pragma unroll
        for (int j = 0; j < 8; j++)
            asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u64 %0, [%1], %2;"
                         : "=l"(kv[j]) : "l"(sin + base + j * 32 + lane), "l"(pc));
#pragma unroll
        for (int j = 0; j < 8; j++) {
            const uint64_t r = mix64(seed + (base + j * 32 + lane) * kGolden + (kv[j] & 1));
            uint16_t x;
            asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u8 %0, [%1], %2;"
                         : "=h"(x) : "l"(buf + __umul64hi(r, F)), "l"(pk));
            v[j] = x;
        }
        uint32_t* st = stage[wq][it & 1];
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");  // buffer free
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 8; j++) st[j * 32 + lane] = v[j] + (uint32_t)kv[j];
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(
                             sout + base),
                         "r"((uint32_t)__cvta_generic_to_shared(st)), "r"(1024u), "l"(pc)
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    if (sink == nullptr) return;
}

// Uniform random gather with a selectable load flavour (DRAM fetch-size experiments).
template <int MODE>
__device__ __forceinline__ uint16_t ld_mode(const uint8_t* p, uint64_t pol) {
    uint16_t x;
    if (MODE == 0) asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u8 %0, [%1], %2;" : "=h"(x) : "l"(p), "l"(pol));
    if (MODE == 1) asm volatile("ld.global.nc.u8 %0, [%1];" : "=h"(x) : "l"(p));
    if (MODE == 2) asm volatile("ld.global.cg.u8 %0, [%1];" : "=h"(x) : "l"(p));
    if (MODE == 3) asm volatile("ld.global.cv.u8 %0, [%1];" : "=h"(x) : "l"(p));
    if (MODE == 4) asm volatile("ld.global.nc.L2::64B.u8 %0, [%1];" : "=h"(x) : "l"(p));
    if (MODE == 5) asm volatile("ld.global.nc.L2::128B.u8 %0, [%1];" : "=h"(x) : "l"(p));
    if (MODE == 6) asm volatile("ld.global.nc.L2::256B.u8 %0, [%1];" : "=h"(x) : "l"(p));
    if (MODE == 7) asm volatile("ld.global.lu.u8 %0, [%1];" : "=h"(x) : "l"(p));
    if (MODE == 8) asm volatile("ld.global.cs.u8 %0, [%1];" : "=h"(x) : "l"(p));
    if (MODE == 9) asm volatile("ld.global.u8 %0, [%1];" : "=h"(x) : "l"(p));
    return x;
}
template <int MODE>
__global__ void __launch_bounds__(256) k_gather_mode(const uint8_t* __restrict__ buf, uint64_t F,
                                                     uint64_t nloads, uint64_t seed, uint32_t* sink) {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * 8;
    uint32_t acc = 0;
    for (uint64_t base = tid * 8; base < nloads; base += stride) {
        uint32_t v[8];
#pragma unroll
        for (int j = 0; j < 8; j++) {
            const uint64_t r = mix64(seed + (base + j) * kGolden);
            v[j] = ld_mode<MODE>(buf + __umul64hi(r, F), pol);
        }
#pragma unroll
        for (int j = 0; j < 8; j++) acc += v[j];
    }
    if (acc == 0x7fffffffu) *sink = acc;
}

// Seeded uniform random ACGT sequence, 2-bit packed MSB-first (ph_gpu.h layout): word w =
// splitmix64 output w of the stream seeded with `seed`.
__global__ void k_gen_dna(uint64_t* out, uint64_t nwords, uint64_t seed) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nwords;
         i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = mix64(seed + (i + 1) * kGolden);
}
// Materialised k-mers (first base in the MSBs), the u64 keys the reference builds over.
__global__ void k_kmers(const uint64_t* __restrict__ seq, uint64_t n_bases, int k, uint64_t* out) {
    const uint64_t n = n_bases - (uint64_t)k + 1, nwords = (n_bases + 31) / 32;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t a = i >> 5;
        const uint32_t o = (uint32_t)(i & 31) * 2;
        const uint64_t wa = seq[a], wb = (o && a + 1 < nwords) ? seq[a + 1] : 0;
        const uint64_t top = o ? (wa << o) | (wb >> (64 - o)) : wa;
        out[i] = k == 32 ? top : top >> (64 - 2 * k);
    }
}

// Config-4 string corpus (same definition as oracle/ph_oracle.c pho_gen_string):
// r0 = mix64(seed + (i+1)*golden); len = 8 + r0 % 57; byte t = 0x21 + mix64(r0 + (t+1)*golden) % 94.
__device__ __forceinline__ uint64_t str_r0(uint64_t i, uint64_t seed) {
    return mix64(seed + (i + 1) * kGolden);
}
__global__ void k_str_lens(uint64_t* lens, uint64_t n, uint64_t seed, uint64_t perm_seed,
                           unsigned h, int permuted) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t src = permuted ? feistel(i, n, perm_seed, h) : i;
        lens[i] = 8 + str_r0(src, seed) % 57;
    }
}
// offsets[i] = start of string i (exclusive scan of lens); writes the bytes of string
// src(i) (identity or the Feistel permutation) at offsets[i].
__global__ void k_str_bytes(const uint64_t* __restrict__ offsets, uint64_t n, uint64_t seed,
                            uint64_t perm_seed, unsigned h, int permuted, uint8_t* out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t src = permuted ? feistel(i, n, perm_seed, h) : i;
        const uint64_t r0 = str_r0(src, seed);
        const uint32_t len = 8 + (uint32_t)(r0 % 57);
        uint8_t* p = out + offsets[i];
        for (uint32_t t = 0; t < len; t++) p[t] = (uint8_t)(0x21 + mix64(r0 + (t + 1) * kGolden) % 94);
    }
}

// Die probe (dual-die L2 study): one thread times a dependent ld.global.cv of the first
// word of each `chunk`-byte block of buf (after a warming pass), recording latency cycles
// and the SM it ran on. Bimodal latencies = near/far home L2.
__global__ void k_die_probe(const uint32_t* buf, uint64_t nchunks, uint32_t chunk_words,
                            uint32_t* lat, uint32_t* smid_out, int passes) {
    __shared__ volatile uint32_t sink_s;
    if (threadIdx.x != 0) return;
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    if (smid_out) smid_out[blockIdx.x] = smid;
    uint32_t v = 1;
    // windows of 4096 chunks (8 MiB at 2 KiB) so the warm pass leaves them L2-resident
    for (uint64_t w0 = 0; w0 < nchunks; w0 += 4096) {
        const uint64_t w1 = w0 + 4096 < nchunks ? w0 + 4096 : nchunks;
        for (int p = 0; p < passes; p++) {
            for (uint64_t c = w0; c < w1; c++) {
                // buf holds ones: (v - 1) == 0 chains each address on the previous load
                const uint32_t* a = buf + c * chunk_words + (v - 1);
                long long t0, t1;
                asm volatile("mov.u64 %0, %%clock64;" : "=l"(t0));
                asm volatile("ld.global.cv.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
                sink_s = v;  // the store waits for the load; clock is read after it issues
                asm volatile("mov.u64 %0, %%clock64;" : "=l"(t1));
                if (p == passes - 1) lat[blockIdx.x * nchunks + c] = (uint32_t)(t1 - t0);
            }
        }
    }
}

// Die-aware gather: a thread on an SM of die d loads random bytes from random chunks of
// list d (chunk_off[d][0..nch[d]) in bytes). sm_die[smid] gives the die of each SM.
// mode 0: die-local lists; mode 1: both lists mixed (control, same footprint).
__global__ void __launch_bounds__(256) k_gather_die(const uint8_t* __restrict__ buf,
                                                    const uint32_t* __restrict__ list0,
                                                    uint32_t n0,
                                                    const uint32_t* __restrict__ list1,
                                                    uint32_t n1, const int8_t* __restrict__ sm_die,
                                                    uint32_t chunk, uint64_t nloads, uint64_t seed,
                                                    int mode, uint32_t* sink) {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    const int d = sm_die[smid];
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * 8;
    uint32_t acc = 0;
    for (uint64_t base = tid * 8; base < nloads; base += stride) {
        uint32_t v[8];
#pragma unroll
        for (int j = 0; j < 8; j++) {
            const uint64_t r = mix64(seed + (base + j) * kGolden);
            int dd = mode == 0 ? d : (int)(r >> 63);
            const uint32_t* L = dd ? list1 : list0;
            const uint32_t n = dd ? n1 : n0;
            const uint32_t c = (uint32_t)__umul64hi(r & 0x7fffffffffffffffull, (uint64_t)n << 1);
            const uint64_t a = (uint64_t)__ldg(L + c) * chunk + ((uint32_t)r % chunk);
            uint16_t x;
            asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u8 %0, [%1], %2;"
                         : "=h"(x) : "l"(buf + a), "l"(pol));
            v[j] = x;
        }
#pragma unroll
        for (int j = 0; j < 8; j++) acc += v[j];
    }
    if (acc == 0x7fffffffu) *sink = acc;
}

__global__ void k_bijection(const uint32_t* __restrict__ out, uint64_t count, uint64_t n,
                            unsigned int* bits, unsigned long long* bad) {
    unsigned long long local_oob = 0, local_dup = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t v = out[i];
        if (v >= n) {
            local_oob++;
            continue;
        }
        const unsigned int m = 1u << (v & 31);
        const unsigned int old = atomicOr(bits + (v >> 5), m);
        if (old & m) local_dup++;
    }
    if (local_oob) atomicAdd(bad, local_oob);
    if (local_dup) atomicAdd(bad + 1, local_dup);
}

int grid(uint64_t count) {
    const uint64_t b = (count + 255) / 256;
    return (int)(b < 148ull * 32 ? (b ? b : 1) : 148ull * 32);
}

}  // namespace

extern "C" {

int phb_gen_queries_perm(uint64_t* d_out, uint64_t start, uint64_t count, uint64_t n,
                         uint64_t gen_seed, uint64_t perm_seed, void* stream) {
    k_gen_perm<<<grid(count), 256, 0, (cudaStream_t)stream>>>(d_out, start, count, n, gen_seed,
                                                             perm_seed, feistel_half_bits(n));
    return (int)cudaGetLastError();
}
int phb_gen_queries_sample(uint64_t* d_out, uint64_t start, uint64_t count, uint64_t n,
                           uint64_t gen_seed, uint64_t sample_seed, void* stream) {
    k_gen_sample<<<grid(count), 256, 0, (cudaStream_t)stream>>>(d_out, start, count, n, gen_seed,
                                                               sample_seed);
    return (int)cudaGetLastError();
}
int phb_gen_corpus(uint64_t* d_out, uint64_t start, uint64_t count, uint64_t gen_seed,
                   void* stream) {
    k_gen_corpus<<<grid(count), 256, 0, (cudaStream_t)stream>>>(d_out, start, count, gen_seed);
    return (int)cudaGetLastError();
}
// host-side twin of k_gen_perm (for building host key arrays without a GPU)
uint64_t phb_perm_key_host(uint64_t i, uint64_t n, uint64_t gen_seed, uint64_t perm_seed) {
    return corpus_u64(feistel(i, n, perm_seed, feistel_half_bits(n)), gen_seed);
}

int phb_gather(const uint8_t* d_buf, uint64_t F, uint64_t nloads, uint64_t seed, int kpt,
               int blocks_per_sm, uint32_t* d_sink, void* stream) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * (blocks_per_sm > 0 ? blocks_per_sm : 8);
    cudaStream_t s = (cudaStream_t)stream;
    switch (kpt) {
        case 1: k_gather<1><<<blocks, 256, 0, s>>>(d_buf, F, nloads, seed, d_sink); break;
        case 4: k_gather<4><<<blocks, 256, 0, s>>>(d_buf, F, nloads, seed, d_sink); break;
        case 16: k_gather<16><<<blocks, 256, 0, s>>>(d_buf, F, nloads, seed, d_sink); break;
        default: k_gather<8><<<blocks, 256, 0, s>>>(d_buf, F, nloads, seed, d_sink); break;
    }
    return (int)cudaGetLastError();
}

int phb_str_lens(uint64_t* d_lens, uint64_t n, uint64_t seed, uint64_t perm_seed, int permuted,
                 void* stream) {
    k_str_lens<<<grid(n), 256, 0, (cudaStream_t)stream>>>(d_lens, n, seed, perm_seed,
                                                        feistel_half_bits(n), permuted);
    return (int)cudaGetLastError();
}
int phb_str_bytes(const uint64_t* d_offsets, uint64_t n, uint64_t seed, uint64_t perm_seed,
                  int permuted, uint8_t* d_out, void* stream) {
    k_str_bytes<<<grid(n), 256, 0, (cudaStream_t)stream>>>(d_offsets, n, seed, perm_seed,
                                                         feistel_half_bits(n), permuted, d_out);
    return (int)cudaGetLastError();
}

int phb_die_probe(const uint32_t* d_buf, uint64_t nchunks, uint32_t chunk_bytes, int blocks,
                  uint32_t* d_lat, uint32_t* d_smid, int passes, void* stream) {
    k_die_probe<<<blocks, 32, 0, (cudaStream_t)stream>>>(d_buf, nchunks, chunk_bytes / 4, d_lat,
                                                        d_smid, passes);
    return (int)cudaGetLastError();
}

int phb_gather_die(const uint8_t* d_buf, const uint32_t* l0, uint32_t n0, const uint32_t* l1,
                   uint32_t n1, const int8_t* sm_die, uint32_t chunk, uint64_t nloads,
                   uint64_t seed, int mode, uint32_t* d_sink, void* stream) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    k_gather_die<<<sms * 8, 256, 0, (cudaStream_t)stream>>>(d_buf, l0, n0, l1, n1, sm_die, chunk,
                                                           nloads, seed, mode, d_sink);
    return (int)cudaGetLastError();
}

int phb_gen_dna(uint64_t* d_out, uint64_t nwords, uint64_t seed, void* stream) {
    k_gen_dna<<<grid(nwords), 256, 0, (cudaStream_t)stream>>>(d_out, nwords, seed);
    return (int)cudaGetLastError();
}
int phb_kmers(const uint64_t* d_seq, uint64_t n_bases, int k, uint64_t* d_out, void* stream) {
    if (n_bases < (uint64_t)k) return 0;
    k_kmers<<<grid(n_bases - k + 1), 256, 0, (cudaStream_t)stream>>>(d_seq, n_bases, k, d_out);
    return (int)cudaGetLastError();
}

int phb_gather_mode(const uint8_t* d_buf, uint64_t F, uint64_t nloads, uint64_t seed, int mode,
                    uint32_t* d_sink, void* stream) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaStream_t s = (cudaStream_t)stream;
    const int g = sms * 8;
#define PHB_M(M) case M: k_gather_mode<M><<<g, 256, 0, s>>>(d_buf, F, nloads, seed, d_sink); break;
    switch (mode) { PHB_M(0) PHB_M(1) PHB_M(2) PHB_M(3) PHB_M(4) PHB_M(5) PHB_M(6) PHB_M(7) PHB_M(8) PHB_M(9) }
#undef PHB_M
    return (int)cudaGetLastError();
}

int phb_gather_skew(const uint8_t* d_buf, uint64_t F_hot, uint64_t F, double p_hot,
                    uint64_t nloads, uint64_t seed, int mode, uint32_t* d_sink, void* stream,
                    const uint64_t* d_sin, uint32_t* d_sout) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const uint32_t ph = (uint32_t)(p_hot * 4294967295.0);
    k_gather_skew<<<sms * 8, 256, 0, (cudaStream_t)stream>>>(d_buf, F_hot, F, ph, nloads, seed,
                                                            mode, d_sink, d_sin, d_sout);
    return (int)cudaGetLastError();
}

// in_words in {0,1,2}, out_bytes in {0,4,8}; d_sin holds nloads*in_words words, d_sout
// nloads*out_bytes bytes. Launches 4 CTAs of 256 threads per SM (pass B's shape).
int phb_port_model(const uint8_t* d_buf, uint64_t F, uint64_t nloads, uint64_t seed, int in_words,
                   int out_bytes, const uint64_t* d_sin, void* d_sout, uint32_t* d_sink,
                   void* stream) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const cudaStream_t s = (cudaStream_t)stream;
#define PH_PORT(I, O)                                                                        \
    if (in_words == I && out_bytes == O) {                                                   \
        k_port<I, O><<<sms * 4, 256, 0, s>>>(d_buf, F, nloads, seed, d_sin, d_sout, d_sink); \
        return (int)cudaGetLastError();                                                      \
    }
    if (in_words == 1 && out_bytes == -4) {  // 4 B out through shared memory + bulk stores
        k_port_bulk<<<sms * 4, 256, 0, s>>>(d_buf, F, nloads, seed, d_sin, (uint32_t*)d_sout, d_sink);
        return (int)cudaGetLastError();
    }
    PH_PORT(1, 42) PH_PORT(1, 44)
    PH_PORT(0, 0) PH_PORT(1, 0) PH_PORT(2, 0) PH_PORT(0, 4) PH_PORT(1, 4) PH_PORT(1, 8) PH_PORT(2, 4) PH_PORT(2, 8)
#undef PH_PORT
    return (int)cudaErrorInvalidValue;
}

// Context-wide L2 knobs for the tuning sweeps (tools/tune.py).
int phb_set_l2_fetch_granularity(int bytes) {
    return (int)cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)bytes);
}
long long phb_get_l2_fetch_granularity() {
    size_t v = 0;
    cudaDeviceGetLimit(&v, cudaLimitMaxL2FetchGranularity);
    return (long long)v;
}
// Persisting-L2 window on `stream` over [ptr, ptr+bytes) with the given hit ratio;
// bytes == 0 clears it.
int phb_set_persist(void* stream, void* ptr, size_t bytes, float hit_ratio, size_t carve) {
    cudaError_t e = cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, carve);
    if (e != cudaSuccess) return (int)e;
    cudaStreamAttrValue a{};
    a.accessPolicyWindow.base_ptr = ptr;
    a.accessPolicyWindow.num_bytes = bytes;
    a.accessPolicyWindow.hitRatio = hit_ratio;
    a.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    a.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    if (bytes == 0) a.accessPolicyWindow.hitProp = cudaAccessPropertyNormal;
    e = cudaStreamSetAttribute((cudaStream_t)stream, cudaStreamAttributeAccessPolicyWindow, &a);
    if (bytes == 0) cudaCtxResetPersistingL2Cache();
    return (int)e;
}
long long phb_max_persist_bytes() {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxPersistingL2CacheSize, 0);
    return v;
}

// bits: ceil(n/32) zeroed u32 words; bad[0] = out-of-range count, bad[1] = duplicates.
int phb_bijection(const uint32_t* d_out, uint64_t count, uint64_t n, unsigned int* d_bits,
                  unsigned long long* d_bad, void* stream) {
    k_bijection<<<grid(count), 256, 0, (cudaStream_t)stream>>>(d_out, count, n, d_bits, d_bad);
    return (int)cudaGetLastError();
}

}  // extern "C"
