// ph_arith.cuh — pure integer arithmetic of the query path, host + device.
//
// Cheaper forms of two pieces of the reference's query arithmetic that give the SAME value:
//
//   bucket = hi64(B * gamma(x))            include/ptrhash/bucket_fn.hpp:66-72 (gamma :18-32)
//   local  = y mod S  (FastModU64::mod)     include/ptrhash/reduce.hpp:38-43
//
// Both are on the FMA pipe in the query kernels (64x64-bit products are four IMAD.WIDE
// each); pass B of the partitioned path is co-limited by that pipe and the L1->XBAR
// request port (profiles/r02_ncu_passes_config3.txt). The forms here need a few 32-bit
// products instead:
//
// * bucket_fast: gamma(x) is bracketed from the top 32 bits of x alone; when the whole
//   bracket maps to one bucket (all but ~B*12/2^32 of the keys, <0.1 % at the configs)
//   that bucket is exact, otherwise the caller computes the exact 64-bit form.
// * mod_fast: y mod S for 2^13 <= S < 2^21 with two 32-bit Barrett steps through
//   2^32 mod S; exact for every y (bounds below), tested exhaustively on the edges and on
//   random words against 128-bit division (tests/cpp/test_arith.cu).
#pragma once

#include <cstdint>

#if defined(__CUDACC__)
#define PH_HD __host__ __device__ __forceinline__
#else
#define PH_HD inline
#endif

namespace phg {

PH_HD uint32_t mulhi32(uint32_t a, uint32_t b) {
#if defined(__CUDA_ARCH__)
    return __umulhi(a, b);
#else
    return (uint32_t)(((uint64_t)a * b) >> 32);
#endif
}

PH_HD uint64_t mulhi64(uint64_t a, uint64_t b) {
#if defined(__CUDA_ARCH__)
    return __umul64hi(a, b);
#else
    return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}

// Bracket of gamma(x) / 2^32 from X = x >> 32 (bucket_fn.hpp:18-32), for the three
// polynomial bucket functions: lo <= gamma(x) / 2^32 < lo + span.
//   linear     gamma = x:                          [X, X + 1)
//   quadratic  gamma = hi64(x*x):   a2 = hi32(X*X), x2 / 2^32 in [a2, a2 + 4)
//   cubic      gamma = floor(floor((x2 + x3)/2) * 255/256) + floor(x/256),
//              a3 = hi32(a2*X), x3 / 2^32 in [a3, a3 + 7); with
//              L2 = floor(((a2>>1) + (a3>>1)) * 255/256) + (X>>8) (each floor loses < 1):
//              gamma / 2^32 in (L2 - 1, L2 + 9)   =>  lo = max(L2 - 1, 0), span = 10
// (x2 >= X^2 and x2 < (X+1)^2 = X^2 + 2X + 1; x3 >= a2*X and
//  x3 < (a2+4)(X+1) = a2*X + a2 + 4X + 4.)
template <int G>
PH_HD uint32_t gamma_bracket(uint32_t X, uint32_t& span) {
    if (G == 0) {
        span = 1;
        return X;
    } else if (G == 1) {
        span = 4;
        return mulhi32(X, X);
    } else {
        const uint32_t a2 = mulhi32(X, X);
        const uint32_t a3 = mulhi32(a2, X);
        const uint32_t L = (a2 >> 1) + (a3 >> 1);                   // <= 2^32 - 3
        const uint32_t L1 = L - (L >> 8) - ((L & 255u) ? 1u : 0u);   // floor(L * 255 / 256)
        const uint32_t L2 = L1 + (X >> 8);
        span = 10;
        return L2 ? L2 - 1 : 0;
    }
}

// bucket = hi64(B * gamma(x)) from the bracket: exact when [lo, lo + span) * B / 2^32
// stays inside one integer, i.e. frac(B * lo / 2^32) + B * span < 2^32. ok = false asks
// the caller for the exact form (probability ~B * span / 2^32). B < 2^32, G in {0,1,2}.
// (L2 + 9 < 2^32 needs gamma < 2^64 - 9 * 2^32, true for any 64-bit gamma; the check
// below rejects every bracket whose image crosses a bucket boundary.)
template <int G>
PH_HD uint32_t bucket_fast(uint32_t X, uint32_t B, bool& ok) {
    uint32_t span;
    const uint32_t lo = gamma_bracket<G>(X, span);
    const uint64_t t = (uint64_t)B * lo;
    ok = (uint64_t)(uint32_t)t + (uint64_t)B * span <= 0xffffffffull;
    return (uint32_t)(t >> 32);
}
template <int G>
constexpr uint32_t gamma_span() {
    return G == 0 ? 1 : G == 1 ? 4 : 10;
}
// The same with the limit hoisted: lim = (2^32 - 1) - B * gamma_span<G>() (negative: the
// fast form never applies).
template <int G>
PH_HD uint32_t bucket_fast_lim(uint32_t X, uint32_t B, int64_t lim, bool& ok) {
    uint32_t span;
    const uint32_t lo = gamma_bracket<G>(X, span);
    const uint64_t t = (uint64_t)B * lo;
    ok = (int64_t)(uint32_t)t <= lim;
    return (uint32_t)(t >> 32);
}
template <int G>
PH_HD int64_t bucket_fast_limit(uint32_t B) {
    return (int64_t)0xffffffffll - (int64_t)B * gamma_span<G>();
}

// Constants of mod_fast for a divisor S (host side, DevIndex::mod_c / mod_m1 / mod_m2).
struct ModFast {
    uint32_t S, nS, c, m1, m2;
    bool ok;  // S in [2^13, 2^21)
};
inline ModFast mod_fast_make(uint64_t S) {
    ModFast m{};
    m.ok = S >= (1u << 13) && S < (1u << 21);
    if (!m.ok) return m;
    m.S = (uint32_t)S;
    m.nS = 0u - (uint32_t)S;
    m.c = (uint32_t)((1ull << 32) % S);
    m.m1 = (uint32_t)((1ull << 32) / S);
    m.m2 = (uint32_t)((1ull << 44) / S);
    return m;
}

// y mod S for 2^13 <= S < 2^21 (= FastModU64::mod(y, S), reduce.hpp:38-43, which is the
// exact remainder for S < 2^32):
//   1. r1 = yh - hi32(yh * m1) * S,  m1 = floor(2^32/S):  r1 = yh mod S or + S  (< 2S)
//   2. t  = r1 * c + yl,             c  = 2^32 mod S:     t == y (mod S), t < 2^44
//   3. q2 = hi32((t >> 12) * m2),    m2 = floor(2^44/S) <= 2^31:  floor(t/S) - 2 <= q2
//      <= floor(t/S), so r = t - q2*S lies in [0, 3S) and fits 32 bits; two conditional
//      subtracts finish it.
// (nS = 2^32 - S: each "x - q*S" is one IMAD x + q*nS mod 2^32.)
PH_HD uint32_t mod_fast(uint64_t y, uint32_t S, uint32_t nS, uint32_t c, uint32_t m1,
                        uint32_t m2) {
    const uint32_t yh = (uint32_t)(y >> 32), yl = (uint32_t)y;
    const uint32_t r1 = yh + mulhi32(yh, m1) * nS;
    const uint64_t t = (uint64_t)r1 * c + yl;
    const uint32_t q2 = mulhi32((uint32_t)(t >> 12), m2);
    uint32_t r = (uint32_t)t + q2 * nS;
    r = r >= S ? r - S : r;
    return r >= S ? r - S : r;
}

}  // namespace phg
