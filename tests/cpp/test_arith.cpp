// Host test of paper_2502_15539_b200/csrc/ph_arith.cuh against the reference's own formulas
// restated with 128-bit integers (bucket_fn.hpp:18-32,66-72; reduce.hpp:38-43, which is the
// exact remainder for S < 2^32). Built and run by tests/test_arith.py (no GPU).
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "ph_arith.cuh"

using u128 = unsigned __int128;
using namespace phg;

static uint64_t mix64(uint64_t z) {  // common.hpp:54-58
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
static uint64_t gamma_ref(int g, uint64_t x) {
    if (g == 0) return x;
    const uint64_t x2 = (uint64_t)(((u128)x * x) >> 64);
    if (g == 1) return x2;
    const uint64_t x3 = (uint64_t)(((u128)x2 * x) >> 64);
    const uint64_t half = (uint64_t)(((u128)x2 + x3) >> 1);
    return (uint64_t)(((u128)half * 255) >> 8) + (x >> 8);
}

int main(int argc, char** argv) {
    const uint64_t N = argc > 1 ? strtoull(argv[1], 0, 10) : 2000000;
    long fails = 0;
    // ---- bucket_fast ----
    const uint32_t Bs[] = {1, 2, 3, 5, 7, 1000, 128206, 189395, 219299, 251383, 1u << 20,
                           (1u << 31) - 1, 0xfffffff0u, 0xffffffffu};
    std::vector<uint64_t> xs;
    for (uint64_t e : {0ull, 1ull, 2ull, 255ull, 256ull, 0xffffffffull, 1ull << 32,
                       (1ull << 32) + 1, 1ull << 63, (1ull << 63) - 1, ~0ull, ~0ull - 1,
                       0xfedcba9876543210ull, 0x9999999999999999ull})
        xs.push_back(e);
    for (uint64_t i = 0; i < N; i++) xs.push_back(mix64(i * 0x9e3779b97f4a7c15ull + 1));
    for (uint64_t X = 0; X < 4096; X++) {  // smallest and largest top words
        xs.push_back(X << 32);
        xs.push_back((X << 32) | 0xffffffffull);
        xs.push_back(~0ull - (X << 32));
    }
    for (int g = 0; g < 3; g++) {
        for (uint32_t B : Bs) {
            uint64_t slow = 0;
            for (uint64_t x : xs) {
                bool ok;
                const uint32_t b = bucket_fast<0>(0, 1, ok);  // (instantiation check)
                (void)b;
                uint32_t got;
                if (g == 0) got = bucket_fast<0>((uint32_t)(x >> 32), B, ok);
                else if (g == 1) got = bucket_fast<1>((uint32_t)(x >> 32), B, ok);
                else got = bucket_fast<2>((uint32_t)(x >> 32), B, ok);
                const uint64_t want = (uint64_t)(((u128)B * gamma_ref(g, x)) >> 64);
                if (!ok) { slow++; continue; }
                if (got != want) {
                    if (fails++ < 10)
                        printf("bucket FAIL g=%d B=%u x=%016llx got %u want %llu\n", g, B,
                               (unsigned long long)x, got, (unsigned long long)want);
                }
            }
            printf("bucket g=%d B=%u: %zu x, exact-path share %.2e\n", g, B, xs.size(),
                   (double)slow / xs.size());
        }
    }
    // ---- mod_fast ----
    std::vector<uint32_t> Ss = {1u << 13, (1u << 13) + 1, 10007, 65535, 65536 + 1, 388501,
                                573922, 664541, 761766, 1000003, (1u << 20) + 7,
                                (1u << 21) - 1, (1u << 21) - 2};
    for (uint64_t i = 0; i < 200; i++) Ss.push_back((1u << 13) + (uint32_t)(mix64(i) % ((1u << 21) - (1u << 13))));
    const uint64_t per = N / 20 + 1000;
    for (uint32_t S : Ss) {
        const ModFast m = mod_fast_make(S);
        if (!m.ok) { printf("mod_fast_make rejected %u\n", S); fails++; continue; }
        auto check = [&](uint64_t y) {
            const uint32_t got = mod_fast(y, m.S, m.nS, m.c, m.m1, m.m2);
            const uint64_t want = y % S;
            if (got != want && fails++ < 10)
                printf("mod FAIL S=%u y=%016llx got %u want %llu\n", S, (unsigned long long)y, got,
                       (unsigned long long)want);
        };
        for (uint64_t y : std::vector<uint64_t>{0ull, 1ull, ~0ull, ~0ull - 1, 1ull << 32, (1ull << 32) - 1,
                           (uint64_t)S, (uint64_t)S - 1, (uint64_t)S + 1, 1ull << 63})
            check(y);
        for (uint64_t k = 1; k < 64; k++) {  // around multiples of S across the range
            const uint64_t q = (~0ull / S) >> k;
            for (int64_t d = -2; d <= 2; d++) check(q * S + d);
            for (int64_t d = -2; d <= 2; d++) check(((~0ull >> k) / S) * S * 1 + d);
        }
        for (uint64_t yh = 0; yh < 64; yh++)  // small/large high words, every residue class edge
            for (uint64_t yl : std::vector<uint64_t>{0ull, 1ull, 0xffffffffull, (uint64_t)S - 1})
                check((yh << 32) | yl), check(((0xffffffffull - yh) << 32) | yl);
        for (uint64_t i = 0; i < per; i++) check(mix64(i ^ ((uint64_t)S << 40)));
    }
    // out-of-range divisors are rejected (the kernels then use the 64-bit form)
    for (uint64_t S : {1ull, 2ull, 8191ull, 1ull << 21, 1ull << 31})
        if (mod_fast_make(S).ok) { printf("mod_fast_make accepted %llu\n", (unsigned long long)S); fails++; }
    printf("%s (%ld failures)\n", fails ? "FAIL" : "OK", fails);
    return fails ? 1 : 0;
}
