// ph_device.cuh — device-side arithmetic of the PtrHash query path (sm_100a).
//
// Bit-exact restatements of the reference's query arithmetic
// (/root/reference/proj, C++), written for the GPU integer pipes:
//   hash_int / hash_pilot        include/ptrhash/hash.hpp:27-32
//   gamma (5 bucket functions)   include/ptrhash/bucket_fn.hpp:18-58, src/bucket_fn.cpp:49-56
//   part_and_bucket              include/ptrhash/bucket_fn.hpp:66-72
//   Reducer / FastModU64         include/ptrhash/reduce.hpp:27-77
//   slot_of / remap_slot         include/ptrhash/index.hpp:91-100
//   CacheLineEF get              include/ptrhash/cacheline_ef.hpp:38-42, :58-73, :86-90
//   plain32 / Elias-Fano get     include/ptrhash/remap.hpp:34-45, src/elias_fano.cpp:51-72
#pragma once

#include <cstdint>

#include "ph_arith.cuh"

#ifndef PH_NO_FAST_BUCKET
#define PH_NO_FAST_BUCKET 1  // 0: bucket_fast with the exact form out of line (A/B builds)
#endif

namespace phg {

constexpr uint64_t kC = 0x517cc1b727220a95ULL;  // hash.hpp:13
constexpr unsigned kFull = 0xffffffffu;

// Everything a query kernel needs, passed by value as a kernel parameter.
struct DevIndex {
    const uint8_t* pilots;        // P*B bytes, byte-identical to the PTRH payload
    const uint8_t* remap;         // CLEF 64-B blocks or plain u32[] (PTRH payload bytes)
    const uint64_t* ef_low;       // Elias-Fano pieces (re-aligned from the payload)
    const uint64_t* ef_high;
    const uint64_t* ef_samples;
    const uint64_t* opt_table;    // 65537-entry optimal-gamma table (host computed)
    uint64_t n, P, S, B, seed;
    uint64_t magic_hi, magic_lo;  // FastModU64::make(S), reduce.hpp:31-36 (kept for reference)
    uint64_t mod_m64;             // floor(2^64 / S) for the device's exact y mod S
    uint64_t hp_base;             // C * (seed & ~0xff): hash_pilot(p) = hp_base + C*((seed^p)&0xff)
    uint32_t seed_lo8;
    // mod_fast constants (ph_arith.cuh) when 2^13 <= S < 2^21 (mod_fast_ok), else the
    // 64-bit form via mod_m64
    uint32_t mod_nS, mod_c, mod_m1, mod_m2;  // mod_nS = -S mod 2^32
    int32_t mod_fast_ok;
    int32_t remap_kind;           // 0 plain32, 1 CacheLineEF, 2 Elias-Fano
    int32_t ef_low_bits;
    int32_t hash_algo;
    // Hot-first pilot layout. The bucket functions put most keys in the
    // first buckets of every part (cubic gamma: the first ~19% of each part's pilots
    // serve ~50% of the queries). The device copy of the pilots stores the first hot_b
    // buckets of every part contiguously ([0, P*hot_b), covered by a persisting L2
    // access-policy window) and the remaining cold_b = B - hot_b buckets after it. It is
    // a permutation of the PTRH pilot bytes; hot_b == B is the file's own layout.
    uint64_t hot_b, cold_b, hot_total;
    uint64_t window_bytes;        // persisting window over the hot region (0 = none)
    float window_hit_ratio;
    int32_t cold_evict_first;     // cold-region pilot loads: 1 = L2::evict_first, 0 = evict_last
    int32_t pilot_evict_normal;   // 1: pilot loads L2::evict_normal instead of evict_last (A/B knob)
    // AES string hash round keys k0/k1 (hash.cpp:116-119) as LE u32 words, host-derived
    uint32_t aes_k0[4], aes_k1[4];
    const uint32_t* aes_tab;      // T0..T3 (4 x 256 words) in global memory (small batches)
};

// Device address of pilots[part*B + bucket] under the hot-first layout.
// P, B < 2^32 (checked at create), so both products are single IMAD.WIDE.U32.
__device__ __forceinline__ uint64_t pilot_offset(const DevIndex& ix, uint32_t part,
                                                 uint32_t bucket) {
    return bucket < (uint32_t)ix.hot_b
               ? (uint64_t)part * (uint32_t)ix.hot_b + bucket
               : ix.hot_total + (uint64_t)part * (uint32_t)ix.cold_b + (bucket - (uint32_t)ix.hot_b);
}

// ---------------------------------------------------------------------------
// cache-policy loads/stores
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
// streamed key: read once, do not keep in L1, evict first from L2
__device__ __forceinline__ uint64_t ld_stream_u64(const uint64_t* p, uint64_t pol) {
    uint64_t v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(pol));
    return v;
}
// the random 1-byte pilot gather: read-only path, keep in L2 ahead of the stream
__device__ __forceinline__ uint32_t ld_gather_u8(const uint8_t* p, uint64_t pol) {
    uint16_t v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.u8 %0, [%1], %2;" : "=h"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ void st_stream(uint32_t* p, uint64_t v) {
    asm volatile("st.global.cs.u32 [%0], %1;" ::"l"(p), "r"((uint32_t)v) : "memory");
}
__device__ __forceinline__ void st_stream(uint64_t* p, uint64_t v) {
    asm volatile("st.global.cs.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// ---------------------------------------------------------------------------
// 64-bit integer helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t mulhi(uint64_t a, uint64_t b) { return __umul64hi(a, b); }

// 32x64 -> 96-bit product: returns hi64(a*b), sets lo = lo64(a*b). Two IMAD.WIDE.U32.
__device__ __forceinline__ uint64_t mul32x64(uint32_t a, uint64_t b, uint64_t& lo) {
    const uint64_t p0 = (uint64_t)a * (uint32_t)b;
    const uint64_t p1 = (uint64_t)a * (uint32_t)(b >> 32);
    const uint64_t mid = p1 + (p0 >> 32);  // < 2^64: no overflow
    lo = (mid << 32) | (uint32_t)p0;
    return mid >> 32;
}

// ((u128)a * b) >> s for 0 < s < 64
__device__ __forceinline__ uint64_t mul_shr(uint64_t a, uint64_t b, int s) {
    return (a * b >> s) | (__umul64hi(a, b) << (64 - s));
}

// ---------------------------------------------------------------------------
// bucket functions gamma, bucket_fn.hpp:18-58
// ---------------------------------------------------------------------------
template <int G>
__device__ __forceinline__ uint64_t gamma(uint64_t x, const uint64_t* __restrict__ opt) {
    if constexpr (G == 0) {  // linear :20
        return x;
    } else if constexpr (G == 1) {  // quadratic :22
        return mulhi(x, x);
    } else if constexpr (G == 2) {  // cubic :27-32: ((x2+x3)>>1)*255>>8 + x>>8, exact
        const uint64_t x2 = mulhi(x, x);
        const uint64_t x3 = mulhi(x2, x);
        // half = floor((x2+x3)/2) from the 65-bit sum (carry into bit 63)
        const uint64_t s = x2 + x3;
        const uint64_t half = (s >> 1) | ((uint64_t)(s < x2) << 63);
        // floor(255*half/256) = half - ceil(half/256)
        return half - (half >> 8) - ((half & 255) != 0) + (x >> 8);
    } else if constexpr (G == 3) {  // skewed :34-39
        constexpr uint64_t SX = 0x9999999999999999ULL;  // floor(3*2^64/5)
        constexpr uint64_t SY = 0x4ccccccccccccccc;     // floor(3*2^64/10)
        if (x < SX) return x >> 1;
        return SY + mul_shr(x - SX, 7, 2);
    } else {  // optimal, bucket_fn.cpp:49-56: table interpolation (table uploaded from host)
        const uint64_t idx = x >> 48;
        const uint64_t frac = x & ((1ULL << 48) - 1);
        const uint64_t lo = __ldg(opt + idx);
        const uint64_t hi = __ldg(opt + idx + 1);
        return lo + mul_shr(hi - lo, frac, 48);
    }
}

// ---------------------------------------------------------------------------
// reduce, reduce.hpp:38-43 / :67-70
// ---------------------------------------------------------------------------
// MF: 1 = mod_fast (the caller checked ix.mod_fast_ok), 0 = the 64-bit form, -1 = decide
// from ix.mod_fast_ok at run time (a uniform branch).
template <bool POW2, int MF = -1>
__device__ __forceinline__ uint64_t reduce(const DevIndex& ix, uint64_t y) {
    if constexpr (POW2) {
        return mulhi(kC, y) & (ix.S - 1);
    } else {
        // FastModU64::mod (reduce.hpp:38-43) is the exact y mod S for S < 2^32 (Lemire's
        // 128-bit-magic bound; verified against 128-bit division in tests/test_oracle.py).
        // Same value, fewer multiplies: q = hi64(y * floor(2^64/S)) is floor(y/S) or one
        // less, so r = y - q*S lies in [0, 2S) and one conditional subtract finishes it.
        // For 2^13 <= S < 2^21 (every config) mod_fast gives the same value with 32-bit
        // products only (ph_arith.cuh); the branch is on a kernel parameter (uniform).
        if (MF == 1 || (MF == -1 && ix.mod_fast_ok))
            return mod_fast(y, (uint32_t)ix.S, ix.mod_nS, ix.mod_c, ix.mod_m1, ix.mod_m2);
        const uint64_t q = mulhi(y, ix.mod_m64);
        uint64_t r = y - q * (uint32_t)ix.S;
        return r >= ix.S ? r - ix.S : r;
    }
}

// bucket = hi64(B * gamma(x)) (bucket_fn.hpp:66-72), B < 2^32. For the polynomial bucket
// functions (linear, quadratic, cubic) bucket_fast brackets gamma from the top word of x
// and is exact for all but ~B*10/2^32 of the keys; those take the 64-bit form out of line.
template <int G>
static __device__ __noinline__ uint32_t bucket_exact(uint64_t x, uint32_t B,
                                                     const uint64_t* __restrict__ opt) {
    uint64_t unused;
    return (uint32_t)mul32x64(B, gamma<G>(x, opt), unused);
}
template <int G, bool FAST = !PH_NO_FAST_BUCKET>
__device__ __forceinline__ uint32_t bucket_of(uint64_t x, uint32_t B,
                                              const uint64_t* __restrict__ opt) {
    if constexpr (G <= 2 && FAST) {
        bool ok;
        const uint32_t b = bucket_fast<G>((uint32_t)(x >> 32), B, ok);
        if (__builtin_expect(ok, 1)) return b;
        return bucket_exact<G>(x, B, opt);
    } else {
        uint64_t unused;
        return (uint32_t)mul32x64(B, gamma<G>(x, opt), unused);
    }
}

__device__ __forceinline__ uint64_t hash_pilot(const DevIndex& ix, uint32_t pilot) {
    // C*(pilot ^ seed) == C*(seed & ~0xff) + C*((seed ^ pilot) & 0xff)  (mod 2^64)
    return ix.hp_base + kC * (uint64_t)((ix.seed_lo8 ^ pilot) & 0xffu);
}

// ---------------------------------------------------------------------------
// remap decodes (rare path: slot >= n)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t select32(uint32_t w, uint32_t rank) {
    return __fns(w, 0, (int)rank + 1);  // rank-th (0-based) set bit
}

// CacheLineEF, cacheline_ef.hpp:86-90; block layout :58-73 (offset u32 LE @0,
// 128-bit mask LE @4, low bytes @20)
__device__ __forceinline__ uint64_t clef_get(const uint8_t* __restrict__ remap, uint64_t idx) {
    const uint32_t blk = (uint32_t)(idx / 44);
    const uint32_t i = (uint32_t)(idx - (uint64_t)blk * 44);
    const uint32_t* w = reinterpret_cast<const uint32_t*>(remap + (uint64_t)blk * 64);
    const uint4 a = __ldg(reinterpret_cast<const uint4*>(w));  // off, m0, m1, m2
    const uint32_t m3 = __ldg(w + 4);
    const uint32_t low = __ldg(remap + (uint64_t)blk * 64 + 20 + i);
    uint32_t r = i, pos;
    const uint32_t c0 = __popc(a.y);
    if (r < c0) {
        pos = select32(a.y, r);
    } else {
        r -= c0;
        const uint32_t c1 = __popc(a.z);
        if (r < c1) {
            pos = 32 + select32(a.z, r);
        } else {
            r -= c1;
            const uint32_t c2 = __popc(a.w);
            pos = (r < c2) ? 64 + select32(a.w, r) : 96 + select32(m3, r - c2);
        }
    }
    return ((uint64_t)a.x << 8) + ((uint64_t)(pos - i) << 8) + low;
}

__device__ __forceinline__ uint32_t select64(uint64_t w, uint32_t rank) {
    const uint32_t lo = (uint32_t)w;
    const uint32_t c = __popc(lo);
    return rank < c ? select32(lo, rank) : 32 + select32((uint32_t)(w >> 32), rank - c);
}

// Elias-Fano, elias_fano.cpp:51-72 (samples pack word<<16 | in-word rank)
__device__ __forceinline__ uint64_t ef_get(const DevIndex& ix, uint64_t i) {
    const uint64_t sample = ix.ef_samples[i / 512];
    uint64_t word = sample >> 16;
    uint32_t want = (uint32_t)(sample & 0xffff) + (uint32_t)(i % 512);
    for (;;) {
        const uint32_t c = __popcll(ix.ef_high[word]);
        if (want < c) break;
        want -= c;
        word++;
    }
    const uint64_t pos = word * 64 + select64(ix.ef_high[word], want);
    const uint32_t l = (uint32_t)ix.ef_low_bits;
    uint64_t low = 0;
    if (l) {
        const uint64_t bitpos = i * l;
        low = ix.ef_low[bitpos / 64] >> (bitpos % 64);
        if (bitpos % 64 + l > 64) low |= ix.ef_low[bitpos / 64 + 1] << (64 - bitpos % 64);
        low &= (1ULL << l) - 1;
    }
    return ((pos - i) << l) | low;
}

// RemapTable::get, remap.hpp:34-45 (kind is warp-uniform)
__device__ __forceinline__ uint64_t remap_get(const DevIndex& ix, uint64_t idx) {
    if (ix.remap_kind == 1) return clef_get(ix.remap, idx);
    if (ix.remap_kind == 0) return __ldg(reinterpret_cast<const uint32_t*>(ix.remap) + idx);
    return ef_get(ix, idx);
}

// The same decode as an out-of-line call, for the query kernels' rare paths: keeps the
// decode's registers out of the hot loop's allocation (occupancy).
static __device__ __noinline__ uint64_t remap_get_call(const uint8_t* remap,
                                                      const uint64_t* ef_low,
                                                      const uint64_t* ef_high,
                                                      const uint64_t* ef_samples, int kind,
                                                      int low_bits, uint64_t idx) {
    DevIndex v;
    v.remap = remap;
    v.ef_low = ef_low;
    v.ef_high = ef_high;
    v.ef_samples = ef_samples;
    v.remap_kind = kind;
    v.ef_low_bits = low_bits;
    return remap_get(v, idx);
}
__device__ __forceinline__ uint64_t remap_get_cold(const DevIndex& ix, uint64_t idx) {
    return remap_get_call(ix.remap, ix.ef_low, ix.ef_high, ix.ef_samples, ix.remap_kind,
                          ix.ef_low_bits, idx);
}

// Warp-cooperative remap of the keys flagged in need[] (slot >= n).
// Entries are ranked across (j, lane) with ballots; lane r of a round decodes
// entry base+r; results return to their owners with shuffles.
template <int KPT, class OutT>
__device__ __forceinline__ void remap_tile(const DevIndex& ix, const bool (&need)[KPT],
                                           uint64_t (&slot)[KPT]) {
    const unsigned lane = threadIdx.x & 31;
    const unsigned lt_mask = (1u << lane) - 1;
    unsigned m[KPT];
    unsigned cum[KPT];
    unsigned total = 0;
#pragma unroll
    for (int j = 0; j < KPT; j++) {
        m[j] = __ballot_sync(kFull, need[j]);
        cum[j] = total;
        total += __popc(m[j]);
    }
    if (total == 0) return;  // warp-uniform
    for (unsigned base = 0; base < total; base += 32) {
        const unsigned r = base + lane;
        // gather the slot of entry r from its owner (j, src)
        uint64_t my = 0;
#pragma unroll
        for (int j = 0; j < KPT; j++) {
            const unsigned cnt = __popc(m[j]);
            const bool mine = r >= cum[j] && r < cum[j] + cnt;
            const unsigned src = mine ? __fns(m[j], 0, (int)(r - cum[j]) + 1) : 0;
            const uint64_t v = __shfl_sync(kFull, slot[j], src & 31);
            if (mine) my = v;
        }
        uint64_t val = 0;
        if (r < total) val = remap_get(ix, my - ix.n);
        // hand results back
#pragma unroll
        for (int j = 0; j < KPT; j++) {
            const unsigned rr = cum[j] + __popc(m[j] & lt_mask);
            const uint64_t v = __shfl_sync(kFull, val, (rr - base) & 31);
            if (need[j] && rr >= base && rr < base + 32) slot[j] = v;
        }
    }
}

}  // namespace phg
