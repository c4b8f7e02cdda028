// ph_query_bytes.cu — string-key query kernel (sm_100a).
//
// Keys are one concatenated byte buffer + u64 offsets[n+1]. Each key is hashed
// with the index's string hash (hash_bytes, /root/reference/proj/src/hash.cpp:159-193):
//   kAes64/kAes128   software AESENC/AESENCLAST rounds (T-tables in shared
//                    memory) reproducing the AES-NI chain of hash.cpp:114-153;
//   kPortable64/128  the folded-multiply hash of hash.cpp:87-104 / :184-190
//                    (kFx64 on bytes also uses it, hash.cpp:162-167).
// then goes through the same slot_of / remap_slot as the u64 path.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>

#include "ph_device.cuh"
#include "ph_kernels.h"

namespace phg {

constexpr uint64_t kP1 = 0x8bb84b93962eacc9ULL;  // hash.cpp:83-85
constexpr uint64_t kP2 = 0x2d358dccaa6c78a5ULL;
constexpr uint64_t kP3 = 0x4b33a62ed433d4a3ULL;
constexpr uint64_t kGolden = 0x9e3779b97f4a7c15ULL;

// AES S-box (FIPS-197), used to fill the shared-memory T-tables.
__constant__ uint8_t c_sbox[256] = {
    0x63, 0x7c, 0x77, 0x7b, 0xf2, 0x6b, 0x6f, 0xc5, 0x30, 0x01, 0x67, 0x2b, 0xfe, 0xd7, 0xab, 0x76,
    0xca, 0x82, 0xc9, 0x7d, 0xfa, 0x59, 0x47, 0xf0, 0xad, 0xd4, 0xa2, 0xaf, 0x9c, 0xa4, 0x72, 0xc0,
    0xb7, 0xfd, 0x93, 0x26, 0x36, 0x3f, 0xf7, 0xcc, 0x34, 0xa5, 0xe5, 0xf1, 0x71, 0xd8, 0x31, 0x15,
    0x04, 0xc7, 0x23, 0xc3, 0x18, 0x96, 0x05, 0x9a, 0x07, 0x12, 0x80, 0xe2, 0xeb, 0x27, 0xb2, 0x75,
    0x09, 0x83, 0x2c, 0x1a, 0x1b, 0x6e, 0x5a, 0xa0, 0x52, 0x3b, 0xd6, 0xb3, 0x29, 0xe3, 0x2f, 0x84,
    0x53, 0xd1, 0x00, 0xed, 0x20, 0xfc, 0xb1, 0x5b, 0x6a, 0xcb, 0xbe, 0x39, 0x4a, 0x4c, 0x58, 0xcf,
    0xd0, 0xef, 0xaa, 0xfb, 0x43, 0x4d, 0x33, 0x85, 0x45, 0xf9, 0x02, 0x7f, 0x50, 0x3c, 0x9f, 0xa8,
    0x51, 0xa3, 0x40, 0x8f, 0x92, 0x9d, 0x38, 0xf5, 0xbc, 0xb6, 0xda, 0x21, 0x10, 0xff, 0xf3, 0xd2,
    0xcd, 0x0c, 0x13, 0xec, 0x5f, 0x97, 0x44, 0x17, 0xc4, 0xa7, 0x7e, 0x3d, 0x64, 0x5d, 0x19, 0x73,
    0x60, 0x81, 0x4f, 0xdc, 0x22, 0x2a, 0x90, 0x88, 0x46, 0xee, 0xb8, 0x14, 0xde, 0x5e, 0x0b, 0xdb,
    0xe0, 0x32, 0x3a, 0x0a, 0x49, 0x06, 0x24, 0x5c, 0xc2, 0xd3, 0xac, 0x62, 0x91, 0x95, 0xe4, 0x79,
    0xe7, 0xc8, 0x37, 0x6d, 0x8d, 0xd5, 0x4e, 0xa9, 0x6c, 0x56, 0xf4, 0xea, 0x65, 0x7a, 0xae, 0x08,
    0xba, 0x78, 0x25, 0x2e, 0x1c, 0xa6, 0xb4, 0xc6, 0xe8, 0xdd, 0x74, 0x1f, 0x4b, 0xbd, 0x8b, 0x8a,
    0x70, 0x3e, 0xb5, 0x66, 0x48, 0x03, 0xf6, 0x0e, 0x61, 0x35, 0x57, 0xb9, 0x86, 0xc1, 0x1d, 0x9e,
    0xe1, 0xf8, 0x98, 0x11, 0x69, 0xd9, 0x8e, 0x94, 0x9b, 0x1e, 0x87, 0xe9, 0xce, 0x55, 0x28, 0xdf,
    0x8c, 0xa1, 0x89, 0x0d, 0xbf, 0xe6, 0x42, 0x68, 0x41, 0x99, 0x2d, 0x0f, 0xb0, 0x54, 0xbb, 0x16};

// The MixColumns∘SubBytes tables T0[x] = (2·S[x], S[x], S[x], 3·S[x]) (rows 0..3, LE) and
// its rotations T1..T3 (by 8/16/24 bits), each held in shared memory 32 times, interleaved
// by lane: every lane reads its own copy, i.e. its own bank, so the 16 lookups of an AES
// round are conflict-free whatever the state bytes are, and a column is four lookups XORed
// with no rotates. S[x] is byte 1 of T0[x] (for AESENCLAST). The four tables (128 KiB) fit
// once per SM, in one 1024-thread CTA (config 4: 9.39 ms against 9.63 with two tables and
// 11.41 with one table at 4 x 256 threads per SM).
// init[len] caches the state after the first AESENC of aes_core for len < kInitLens: it
// depends only on (len, seed), hash.cpp:120-122.
constexpr uint32_t kInitLens = 256;
// Four tables in two 64 KiB halves: entry x of table t for lane l sits at byte
// (t>>1)*64 KiB + x*256 + (t&1)*128 + l*4 from the table base, which is placed at shared
// address kTabBase (64 KiB-aligned): one PRMT then forms the whole shared address from the
// state word and lw = kTabBase + l*4 (byte K of the state word into byte 1; bytes 0, 2, 3
// from lw), and the table is the LDS immediate -- two instructions per lookup.
constexpr uint32_t kTabBase = 0x10000;
struct AesTables {
    uint32_t t[4 * 256 * 32];  // 128 KiB
};

__device__ __forceinline__ uint8_t xtime(uint8_t a) {
    return (uint8_t)((a << 1) ^ ((a & 0x80) ? 0x1b : 0));
}

__device__ __forceinline__ uint32_t t0_entry(int x) {
    const uint8_t s = c_sbox[x];
    const uint8_t s2 = xtime(s), s3 = (uint8_t)(s2 ^ s);
    return (uint32_t)s2 | ((uint32_t)s << 8) | ((uint32_t)s << 16) | ((uint32_t)s3 << 24);
}

__device__ void fill_tables(AesTables& T) {
    for (int e = threadIdx.x; e < 4 * 256 * 32; e += blockDim.x) {
        const int t = e >> 13, x = (e >> 5) & 255, l = e & 31;
        const uint32_t v = t0_entry(x);
        T.t[((t >> 1) << 14) + (x << 6) + ((t & 1) << 5) + l] = __funnelshift_l(v, v, 8 * t);
    }
}
// Lookup of table TABLE at byte K of w in this lane's copy (tb = kTabBase + lane*4).
struct SmemLook {
    uint32_t tb;
    template <int K, int TABLE>
    __device__ __forceinline__ uint32_t get(uint32_t w) const {
        uint32_t a, v;
        asm("prmt.b32 %0, %1, %2, %3;" : "=r"(a) : "r"(w), "r"(tb), "n"(0x7604 | (K << 4)));
        asm volatile("ld.shared.u32 %0, [%1+%2];" : "=r"(v)
                     : "r"(a), "n"((TABLE >> 1) * 65536 + (TABLE & 1) * 128));
        return v;
    }
};
// The same four tables, one copy each, staged in shared memory by a small launch (few lanes,
// so bank conflicts do not matter; one round trip to L2 for the whole 4 KiB instead of one
// per dependent AES round).
struct FlatLook {
    const uint32_t* tab;  // shared memory
    template <int K, int TABLE>
    __device__ __forceinline__ uint32_t get(uint32_t w) const {
        return tab[TABLE * 256 + ((w >> (8 * K)) & 255)];
    }
};
__device__ __forceinline__ void stage_aes_tab(uint32_t* dst, const uint32_t* __restrict__ src) {
    for (uint32_t i = threadIdx.x; i < 1024 / 4; i += blockDim.x)
        reinterpret_cast<uint4*>(dst)[i] = __ldg(reinterpret_cast<const uint4*>(src) + i);
}

__device__ __forceinline__ void prefetch_l2(const void* p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// 16-byte load of key bytes: read-only global path, or (GEN) a generic load, for keys
// staged in shared memory (k_index_bytes_one).
template <bool GEN>
__device__ __forceinline__ uint4 ldq(const uint4* p) {
    if constexpr (GEN) return *p;
    else return __ldg(p);
}

// state: 4 little-endian u32 columns (byte 4c+r = row r of column c), i.e. the
// in-memory byte order of the __m128i in hash.cpp. AESENC = ShiftRows,
// SubBytes, MixColumns, AddRoundKey (Intel semantics).
template <class L>
__device__ __forceinline__ void aesenc(uint32_t (&s)[4], const uint32_t (&k)[4], const L& T) {
    uint32_t o[4];
#pragma unroll
    for (int c = 0; c < 4; c++) {
        const uint32_t a0 = T.template get<0, 0>(s[c]);
        const uint32_t a1 = T.template get<1, 1>(s[(c + 1) & 3]);
        const uint32_t a2 = T.template get<2, 2>(s[(c + 2) & 3]);
        const uint32_t a3 = T.template get<3, 3>(s[(c + 3) & 3]);
        o[c] = a0 ^ a1 ^ a2 ^ a3 ^ k[c];
    }
#pragma unroll
    for (int c = 0; c < 4; c++) s[c] = o[c];
}
template <class L>
__device__ __forceinline__ void aesenclast(uint32_t (&s)[4], const uint32_t (&k)[4], const L& T) {
    uint32_t o[4];
#pragma unroll
    for (int c = 0; c < 4; c++) {
        const uint32_t a0 = T.template get<0, 0>(s[c]), a1 = T.template get<1, 0>(s[(c + 1) & 3]);
        const uint32_t a2 = T.template get<2, 0>(s[(c + 2) & 3]), a3 = T.template get<3, 0>(s[(c + 3) & 3]);
        // S[x] is byte 1 of T0[x]: gather byte 1 of a0..a3 into bytes 0..3
        uint32_t lo, hi, v;
        asm("prmt.b32 %0, %1, %2, 0x0051;" : "=r"(lo) : "r"(a0), "r"(a1));  // bytes 0,1
        asm("prmt.b32 %0, %1, %2, 0x5100;" : "=r"(hi) : "r"(a2), "r"(a3));  // bytes 2,3
        asm("prmt.b32 %0, %1, %2, 0x7610;" : "=r"(v) : "r"(lo), "r"(hi));
        o[c] = v ^ k[c];
    }
#pragma unroll
    for (int c = 0; c < 4; c++) s[c] = o[c];
}

// Bytes [sh, sh+16) of the 32-byte concatenation lo|hi as 4 LE words, zero from byte
// `avail` on (avail < 16: the zero-padded tail block): a two-level select on the word
// shift and one funnel shift per word.
__device__ __forceinline__ void realign16(const uint4& lo, const uint4& hi, uint32_t sh,
                                          uint32_t avail, uint32_t (&w)[4]) {
    const uint32_t r[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
    uint32_t s2[7], a[5];
    const bool w2 = sh & 8, w1 = sh & 4;
#pragma unroll
    for (int t = 0; t < 7; t++) s2[t] = w2 ? (t + 2 < 8 ? r[t + 2] : 0) : r[t];
#pragma unroll
    for (int t = 0; t < 5; t++) a[t] = w1 ? s2[t + 1] : s2[t];
    const uint32_t rb = (sh & 3) * 8;
#pragma unroll
    for (int t = 0; t < 4; t++) w[t] = __funnelshift_r(a[t], a[t + 1], rb);
    if (avail < 16) {
#pragma unroll
        for (int t = 0; t < 4; t++) {
            const int keep = (int)avail - 4 * t;  // bytes to keep in word t
            if (keep <= 0) w[t] = 0;
            else if (keep < 4) w[t] &= (1u << (8 * keep)) - 1;
        }
    }
}

// Loads min(avail,16) bytes at base+off as 4 LE words, zero past `avail`, with at most
// two aligned 16-byte loads. Only aligned 16-byte granules that hold at least one
// requested byte are read, so no access leaves the granules covering the key.
template <bool GEN>
__device__ __forceinline__ void load16(const uint8_t* __restrict__ base, uint64_t off,
                                       uint32_t avail, uint32_t (&w)[4]) {
    const uintptr_t addr = reinterpret_cast<uintptr_t>(base + off);
    const uint4* p = reinterpret_cast<const uint4*>(addr & ~uintptr_t{15});
    const uint32_t sh = (uint32_t)(addr & 15);
    const uint32_t nb = avail < 16 ? avail : 16;
    const uint4 lo = ldq<GEN>(p);
    const uint4 hi = (sh + nb > 16) ? ldq<GEN>(p + 1) : make_uint4(0, 0, 0, 0);
    realign16(lo, hi, sh, avail, w);
}

__device__ __forceinline__ uint64_t mum(uint64_t a, uint64_t b) {  // hash.cpp:53-56
    return (a * b) ^ __umul64hi(a, b);
}

__device__ __forceinline__ uint64_t w64(const uint32_t (&w)[4], int i) {
    return (uint64_t)w[2 * i] | ((uint64_t)w[2 * i + 1] << 32);
}

// portable_hash64, hash.cpp:87-104 (read_tail :71-81)
template <bool GEN>
__device__ uint64_t portable_hash64(const uint8_t* __restrict__ data, uint64_t off, uint32_t len,
                                    uint64_t seed) {
    uint64_t acc = seed ^ mum((uint64_t)len ^ kP1, seed ^ kP2);
    uint32_t i = 0;
    uint32_t w[4];
    while (i + 16 <= len) {
        load16<GEN>(data, off + i, 16, w);
        acc = mum(w64(w, 0) ^ kP1, w64(w, 1) ^ acc);
        i += 16;
    }
    uint64_t a = 0, b = 0;
    const uint32_t rem = len - i;
    if (rem > 0) {
        load16<GEN>(data, off + i, rem, w);  // the remaining 1..15 bytes, zero padded
        auto tail = [&](uint32_t start, uint32_t m) -> uint64_t {  // read_tail(p+start, m)
            auto byte_at = [&](uint32_t q) -> uint64_t { return (w[q >> 2] >> (8 * (q & 3))) & 0xff; };
            if (m >= 4) {
                uint64_t lo = 0, hi = 0;
                for (int t = 0; t < 4; t++) {
                    lo |= byte_at(start + t) << (8 * t);
                    hi |= byte_at(start + m - 4 + t) << (8 * t);
                }
                return lo | (hi << 32);
            }
            return byte_at(start) | (byte_at(start + (m >> 1)) << 8) | (byte_at(start + m - 1) << 16);
        };
        if (rem > 8) {
            a = w64(w, 0);
            b = tail(8, rem - 8);
        } else {
            a = tail(0, rem);
        }
    }
    acc = mum(a ^ kP2 ^ (uint64_t)len, b ^ acc ^ kP3);
    return mum(acc, acc ^ kP1);
}

__device__ __forceinline__ uint64_t mix64(uint64_t z) {  // common.hpp:54-58
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

__device__ __forceinline__ void set128(uint32_t (&s)[4], uint64_t hi, uint64_t lo) {
    s[0] = (uint32_t)lo;
    s[1] = (uint32_t)(lo >> 32);
    s[2] = (uint32_t)hi;
    s[3] = (uint32_t)(hi >> 32);
}

// aes_core + aes_hash, hash.cpp:114-153. k0/k1 come precomputed from the host (they depend
// only on the seed, hash.cpp:116-119); the first round comes from the init table. The
// zero-padded tail block (buf[15] ^= len - i) is the last iteration of the block loop, so a
// key takes exactly ceil(len/16) absorbing rounds.
template <class L, bool GEN, bool INIT>
__device__ __forceinline__ void aes_hash(const uint8_t* __restrict__ data, uint64_t off, uint32_t len,
                         uint64_t seed, bool wide, const DevIndex& ix, uint32_t init_s,
                         const L& tb, uint64_t& hi, uint64_t& lo) {
    const uint32_t k0[4] = {ix.aes_k0[0], ix.aes_k0[1], ix.aes_k0[2], ix.aes_k0[3]};
    const uint32_t k1[4] = {ix.aes_k1[0], ix.aes_k1[1], ix.aes_k1[2], ix.aes_k1[3]};
    uint32_t s[4], w[4];
    if (INIT && len < kInitLens) {  // init: the table's shared-window address
        asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(s[0]), "=r"(s[1]), "=r"(s[2]), "=r"(s[3])
                     : "r"(init_s + len * 16));
    } else {
        set128(s, (uint64_t)len * kC, seed ^ (uint64_t)len);
        aesenc(s, k0, tb);
    }
    // The key's bytes arrive as aligned 16-byte granules g0..gl, prefetched one block ahead
    // (block b needs granules b and b+1; granule b+2 is loaded while block b is hashed), and
    // are realigned with a two-level word select and one funnel shift per word. No granule
    // past gl is read, i.e. no access leaves the granules covering the key. Blocks below the
    // warp's smallest full-block count skip the tail mask (a warp-uniform test); the mask is
    // branch-free (one clamped funnel shift per word).
    const uint32_t nblk = (len + 15) >> 4;
    const uintptr_t a0 = reinterpret_cast<uintptr_t>(data + off);
    const uint4* gp = reinterpret_cast<const uint4*>(a0 & ~uintptr_t{15});
    const uint32_t sh = (uint32_t)(a0 & 15);
    const uint32_t gl = len ? (sh + len - 1) >> 4 : 0;
    const uint32_t nmin = __reduce_min_sync(__activemask(), len >> 4);
    const uint4 zero = make_uint4(0, 0, 0, 0);
    uint4 cur = nblk ? ldq<GEN>(gp) : zero;
    uint4 nxt = gl >= 1 ? ldq<GEN>(gp + 1) : zero;
    for (uint32_t b = 0; b < nblk; b++) {
        const uint4 nn = b + 2 <= gl ? ldq<GEN>(gp + b + 2) : zero;  // prefetch
        realign16(cur, nxt, sh, 16, w);
        if (b >= nmin) {  // this lane may be in its zero-padded tail block
            const uint32_t rem = len - (b << 4);
            const int base = 32 - 8 * (int)rem;  // word t keeps rem - 4t bytes
#pragma unroll
            for (int t = 0; t < 4; t++)
                w[t] &= __funnelshift_rc(0xffffffffu, 0u, (uint32_t)max(base + 32 * t, 0));
            if (rem < 16) w[3] ^= rem << 24;  // buf[15] ^= len - i
        }
#pragma unroll
        for (int c = 0; c < 4; c++) s[c] ^= w[c];
        aesenc(s, k1, tb);
        cur = nxt;
        nxt = nn;
    }
    aesenc(s, k0, tb);
    aesenc(s, k1, tb);
    aesenclast(s, k0, tb);
    const uint64_t l = (uint64_t)s[0] | ((uint64_t)s[1] << 32);
    const uint64_t h = (uint64_t)s[2] | ((uint64_t)s[3] << 32);
    if (!wide) {
        hi = lo = h ^ (l * kC);
    } else {
        hi = h;
        lo = l;
    }
}

// Keys per warp batch. A warp ranks its batch by block count ceil(len/16) (a counting sort
// by ballots) and hashes the keys in that order, 32 at a time, so the lanes of a round run
// the same number of rounds; outputs go back to their input positions.
constexpr int kBatchPer = 4;
constexpr int kBatch = 32 * kBatchPer;
#ifndef PH_STR_THREADS
#define PH_STR_THREADS 1024  // one CTA per SM (registers), one copy of the tables per SM
#endif
constexpr int kBytesThreads = PH_STR_THREADS;
constexpr int kBytesWarps = kBytesThreads / 32;
constexpr uint32_t kClasses = 8;  // block counts 0..6, and 7 for >= 7 blocks

// hash_bytes (hash.cpp:159-193) of the key at data[o0, o1) with the index's string hash.
template <bool GEN = false, bool INIT = false, class L>
__device__ __forceinline__ void hash_key(const uint8_t* __restrict__ data, uint64_t o0,
                                         uint64_t o1, const DevIndex& ix, uint32_t init_s,
                                         const L& look, uint64_t& hi, uint64_t& lo) {
    const int algo = ix.hash_algo;
    const uint32_t len = (uint32_t)(o1 - o0);
    if (algo == 1 || algo == 2) {
        aes_hash<L, GEN, INIT>(data, o0, len, ix.seed, algo == 2, ix, init_s, look, hi, lo);
    } else if (algo == 4) {
        hi = portable_hash64<GEN>(data, o0, len, ix.seed ^ kP3);
        lo = portable_hash64<GEN>(data, o0, len, mix64(ix.seed) + kGolden);
    } else {
        hi = lo = portable_hash64<GEN>(data, o0, len, ix.seed);
    }
}

// part_and_bucket (bucket_fn.hpp:66-72) of a hashed key and its pilot gather, issued
// without waiting (FAST: the bracketed bucket form, ph_arith.cuh).
template <int G, bool FAST, bool HOTF = true>
__device__ __forceinline__ uint32_t locate(const DevIndex& ix, bool valid, uint64_t hi,
                                           uint32_t& part, uint64_t pol_keep, uint64_t pol_cold) {
    uint64_t x;
    part = (uint32_t)mul32x64((uint32_t)ix.P, hi, x);  // P, B < 2^32 (create)
    const uint32_t bucket = bucket_of<G, FAST>(x, (uint32_t)ix.B, ix.opt_table);
    if constexpr (!HOTF)  // the file's own layout (hot_b == B)
        return valid ? ld_gather_u8(ix.pilots + ((uint64_t)part * (uint32_t)ix.B + bucket), pol_keep)
                     : 0;
    const bool hot = bucket < ix.hot_b;
    return valid ? ld_gather_u8(ix.pilots + pilot_offset(ix, part, bucket),
                                (hot || !ix.cold_evict_first) ? pol_keep : pol_cold)
                 : 0;
}

// slot_of + remap_slot (index.hpp:91-100) from the key's part, low hash word and pilot,
// stored to *dst; warp-collective (the rare remap decodes run convergently), `valid` masks
// the lanes without a key.
template <bool POW2, int MF, class OutT>
__device__ __forceinline__ void finish(const DevIndex& ix, bool valid, uint32_t part,
                                       uint64_t lo, uint32_t pilot, int minimal, OutT* dst) {
    uint64_t slot = (uint64_t)part * (uint32_t)ix.S + reduce<POW2, MF>(ix, lo ^ hash_pilot(ix, pilot));
    if (minimal) {
        const bool need = valid && slot >= ix.n;
        if (__any_sync(kFull, need)) {
            // rare path: every flagged lane decodes (one convergent round per warp)
            uint64_t v = 0;
            if (need) v = remap_get(ix, slot - ix.n);
            if (need) slot = v;
        }
    }
    if (valid) st_stream(dst, slot);
}

template <int G, bool POW2, class OutT>
__device__ __forceinline__ void answer_key(const DevIndex& ix, bool valid, uint64_t hi,
                                           uint64_t lo, int minimal, OutT* dst,
                                           uint64_t pol_keep, uint64_t pol_cold) {
    uint32_t part;
    const uint32_t pilot = locate<G, false>(ix, valid, hi, part, pol_keep, pol_cold);
    finish<POW2, -1>(ix, valid, part, lo, pilot, minimal, dst);
}

// Batches of at most 32 keys (single-key index(), tiny batches): one warp, one key per lane,
// AES T-tables read from global memory (4 KiB, L1-resident) instead of filling the 128 KiB
// shared-memory copies, which would dominate a one-key launch.
template <int G, bool POW2, class OutT>
__global__ void __launch_bounds__(32) k_query_bytes_small(const DevIndex ix,
                                                          const uint8_t* __restrict__ data,
                                                          const uint64_t* __restrict__ offsets,
                                                          uint64_t base_off, OutT* __restrict__ out,
                                                          uint64_t nkeys, int minimal) {
    __shared__ __align__(16) uint32_t tab[1024];
    const unsigned lane = threadIdx.x;
    const bool valid = lane < nkeys;
    if (ix.hash_algo == 1 || ix.hash_algo == 2) stage_aes_tab(tab, ix.aes_tab);
    __syncwarp();
    uint64_t hi = 0, lo = 0;
    if (valid)
        hash_key(data, offsets[lane] - base_off, offsets[lane + 1] - base_off, ix, 0u,
                 FlatLook{tab}, hi, lo);
    answer_key<G, POW2>(ix, valid, hi, lo, minimal, out + lane, policy_evict_last(),
                        policy_evict_first());
}

// index(string_view) for one key of at most kOneKeyBytes bytes (ph_gpu_index_bytes): the key
// travels in the launch parameters, so the kernel reads nothing from the host; it is staged
// in shared memory and hashed by lane 0.
constexpr uint32_t kOneKeyBytes = 256;  // (launch-parameter bytes cost launch latency)
struct OneKey {
    uint4 bytes[kOneKeyBytes / 16];
    uint64_t len;
};
template <int G, bool POW2>
__global__ void __launch_bounds__(32) k_index_bytes_one(const DevIndex ix, const OneKey key,
                                                        uint64_t* __restrict__ out, int minimal) {
    __shared__ __align__(16) uint4 kb[kOneKeyBytes / 16];
    __shared__ __align__(16) uint32_t tab[1024];
    const unsigned lane = threadIdx.x;
    if (ix.hash_algo == 1 || ix.hash_algo == 2) stage_aes_tab(tab, ix.aes_tab);
    for (uint32_t i = lane; i < (uint32_t)(key.len + 15) / 16; i += 32) kb[i] = key.bytes[i];
    __syncwarp();
    uint64_t hi = 0, lo = 0;
    if (lane == 0)
        hash_key<true>(reinterpret_cast<const uint8_t*>(kb), 0, key.len, ix, 0u,
                       FlatLook{tab}, hi, lo);
    answer_key<G, POW2>(ix, lane == 0, hi, lo, minimal, out, policy_evict_last(),
                        policy_evict_first());
}

// Dynamic shared memory of k_query_bytes: BytesLow from the start of the window, the AES
// tables at shared address kTabBase (so the allocation spans kTabBase + 128 KiB minus the
// window's start; BytesLow must end below kTabBase, checked at run time).
struct BytesLow {
    uint4 init[kInitLens];                  // states after the first AESENC, by length
    uint64_t off[kBytesWarps][kBatch + 1];  // each warp batch's offsets
    uint8_t perm[kBytesWarps][kBatch];      // the batch in block-count order
};
constexpr size_t kBytesSmem = kTabBase + sizeof(AesTables);  // 192 KiB

template <int G, bool POW2, class OutT, int MF, bool HOTF>
__global__ void __launch_bounds__(kBytesThreads, 1) k_query_bytes(const DevIndex ix,
                                                     const uint8_t* __restrict__ data,
                                                     const uint64_t* __restrict__ offsets,
                                                     uint64_t base_off, OutT* __restrict__ out, uint64_t nkeys,
                                                     int minimal) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    const uint32_t win = (uint32_t)__cvta_generic_to_shared(smem_raw);
    if (win + sizeof(BytesLow) > kTabBase) __trap();  // (the window starts at <= 1 KiB)
    BytesLow& SM = *reinterpret_cast<BytesLow*>(smem_raw);
    AesTables& T = *reinterpret_cast<AesTables*>(smem_raw + (kTabBase - win));
    auto& s_off = SM.off;
    auto& s_perm = SM.perm;
    const int algo = ix.hash_algo;
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1;
    const SmemLook tb{kTabBase + lane * 4};
    const uint32_t init_s = (uint32_t)__cvta_generic_to_shared(SM.init);
    if (algo == 1 || algo == 2) {
        fill_tables(T);
        __syncthreads();
        const uint32_t k0[4] = {ix.aes_k0[0], ix.aes_k0[1], ix.aes_k0[2], ix.aes_k0[3]};
        for (uint32_t len = threadIdx.x; len < kInitLens; len += blockDim.x) {
            uint32_t st[4];
            set128(st, (uint64_t)len * kC, ix.seed ^ (uint64_t)len);  // hash.cpp:120-122
            aesenc(st, k0, tb);
            SM.init[len] = make_uint4(st[0], st[1], st[2], st[3]);
        }
        __syncthreads();
    }
    const uint64_t pol_keep = policy_evict_last();
    const uint64_t pol_cold = policy_evict_first();
    const uint64_t nwarps = (uint64_t)gridDim.x * kBytesWarps;
    uint64_t* so = s_off[warp];
    uint8_t* sp = s_perm[warp];
    for (uint64_t base = (blockIdx.x * (uint64_t)kBytesWarps + warp) * kBatch; base < nkeys;
         base += nwarps * kBatch) {
        const uint32_t cnt = (uint32_t)(nkeys - base < (uint64_t)kBatch ? nkeys - base : kBatch);
        // offsets[base .. base+cnt] into shared memory (coalesced)
#pragma unroll
        for (int r = 0; r < kBatchPer; r++) {
            const uint32_t e = r * 32 + lane;
            if (e <= cnt) so[e] = __ldg(offsets + base + e);
        }
        if (lane == 0 && cnt == kBatch) so[kBatch] = __ldg(offsets + base + kBatch);
        __syncwarp();
        // The batch's key bytes are one contiguous span (~4.6 KB at config 4): touch all of
        // its lines now (L2 prefetch), so the keys hashed later in the batch find them there.
        {
            const uintptr_t lo = reinterpret_cast<uintptr_t>(data + (so[0] - base_off)) & ~uintptr_t{127};
            const uintptr_t hi = reinterpret_cast<uintptr_t>(data + (so[cnt] - base_off));
            for (uintptr_t a = lo + lane * 128; a < hi; a += 32 * 128)
                prefetch_l2(reinterpret_cast<const void*>(a));
        }
        // counting sort of the batch by block count (invalid slots last)
        uint32_t cls[kBatchPer];
#pragma unroll
        for (int r = 0; r < kBatchPer; r++) {
            const uint32_t e = r * 32 + lane;
            const uint64_t len = e < cnt ? so[e + 1] - so[e] : 0;
            const uint64_t nb = (len + 15) >> 4;
            cls[r] = e < cnt ? (nb < kClasses - 1 ? (uint32_t)nb : kClasses - 1) : kClasses;
        }
        uint32_t present = 0;  // classes that occur in the batch (usually 4-5 of 9)
#pragma unroll
        for (int r = 0; r < kBatchPer; r++) present |= 1u << cls[r];
        present = __reduce_or_sync(kFull, present);
        uint32_t run = 0;
        while (present) {
            const uint32_t c = __ffs(present) - 1;
            present &= present - 1;
#pragma unroll
            for (int r = 0; r < kBatchPer; r++) {
                const unsigned m = __ballot_sync(kFull, cls[r] == c);
                if (cls[r] == c) sp[run + __popc(m & lt)] = (uint8_t)(r * 32 + lane);
                run += __popc(m);
            }
        }
        __syncwarp();
        // hash the batch's keys 32 at a time; each key's pilot gather is issued as soon as its
        // hash is known and the key is finished one round later, so the gather overlaps the
        // next key's hashing (one copy of the hash code: the loop is not unrolled)
        uint32_t pe = 0xffffffffu, ppart = 0, ppilot = 0;
        uint64_t plo = 0;
#pragma unroll 1
        for (int q = 0; q <= kBatchPer; q++) {
            uint32_t e = 0xffffffffu, part = 0, pilot = 0;
            uint64_t lo = 0;
            if (q < kBatchPer) {  // (warp-uniform)
                e = sp[q * 32 + lane];
                const bool valid = e < cnt;
                uint64_t hi = 0;
                if (valid)
                    hash_key<false, true>(data, so[e] - base_off, so[e + 1] - base_off, ix,
                                          init_s, tb, hi, lo);
                pilot = locate<G, true, HOTF>(ix, valid, hi, part, pol_keep, pol_cold);
            }
            if (q > 0) finish<POW2, MF>(ix, pe < cnt, ppart, plo, ppilot, minimal, out + base + pe);
            pe = e;
            ppart = part;
            ppilot = pilot;
            plo = lo;
        }
        __syncwarp();  // s_off / s_perm are rewritten by the next batch
    }
}

// Construction of a string-key index (ph_builder.cu): hash_bytes(key, seed).lo of every key
// (hash.cpp:159-193; what build(span<const std::string>) feeds run_attempt<H64>,
// construction.cpp:159-171), written as its pre-image under the integer hash,
// out[i] = Cinv * lo ^ seed, so that the u64 build front (C * (out[i] ^ seed) == lo) sorts
// and searches exactly the string hashes. One key per thread; the AES tables as in
// k_query_bytes. Only ix.seed, ix.hash_algo and the AES round keys of ix are used.
__global__ void __launch_bounds__(kBytesThreads, 1) k_hash_bytes(const DevIndex ix,
                                                                  const uint8_t* __restrict__ data,
                                                                  const uint64_t* __restrict__ offsets,
                                                                  uint64_t* __restrict__ out,
                                                                  uint64_t nkeys, uint64_t cinv) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    const uint32_t win = (uint32_t)__cvta_generic_to_shared(smem_raw);
    if (win + sizeof(BytesLow) > kTabBase) __trap();
    BytesLow& SM = *reinterpret_cast<BytesLow*>(smem_raw);
    AesTables& T = *reinterpret_cast<AesTables*>(smem_raw + (kTabBase - win));
    const unsigned lane = threadIdx.x & 31;
    const SmemLook tb{kTabBase + lane * 4};
    const uint32_t init_s = (uint32_t)__cvta_generic_to_shared(SM.init);
    if (ix.hash_algo == 1 || ix.hash_algo == 2) {
        fill_tables(T);
        __syncthreads();
        const uint32_t k0[4] = {ix.aes_k0[0], ix.aes_k0[1], ix.aes_k0[2], ix.aes_k0[3]};
        for (uint32_t len = threadIdx.x; len < kInitLens; len += blockDim.x) {
            uint32_t st[4];
            set128(st, (uint64_t)len * kC, ix.seed ^ (uint64_t)len);  // hash.cpp:120-122
            aesenc(st, k0, tb);
            SM.init[len] = make_uint4(st[0], st[1], st[2], st[3]);
        }
        __syncthreads();
    }
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nkeys;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t hi, lo;
        hash_key<false, true>(data, __ldg(offsets + i), __ldg(offsets + i + 1), ix, init_s, tb, hi, lo);
        out[i] = (cinv * lo) ^ ix.seed;
    }
}

cudaError_t launch_hash_bytes(const DevIndex& ix, const uint8_t* bytes, const uint64_t* offsets,
                              uint64_t* out, uint64_t n, uint64_t cinv, cudaStream_t s, int sms) {
    if (n == 0) return cudaSuccess;
    constexpr size_t smem = kBytesSmem;
    cudaError_t e = cudaFuncSetAttribute(k_hash_bytes, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const uint64_t want = (n + kBytesThreads - 1) / kBytesThreads;
    const int blocks = (int)(want < (uint64_t)sms ? want : (uint64_t)sms);
    k_hash_bytes<<<blocks, kBytesThreads, smem, s>>>(ix, bytes, offsets, out, n, cinv);
    note_launch();
    return cudaGetLastError();
}

template <int G, bool POW2, class OutT>
static cudaError_t launch_b(const DevIndex& ix, const uint8_t* d, const uint64_t* o,
                            uint64_t bo, void* out, uint64_t n, int minimal, cudaStream_t s, int sms) {
    if (n <= 32) {
        const cudaError_t e = launch_ex(ix, k_query_bytes_small<G, POW2, OutT>, 1, 32, s, ix, d, o,
                                        bo, static_cast<OutT*>(out), n, minimal);
        note_launch();
        return e;
    }
    const bool hotf = ix.hot_b < ix.B;
    void (*kern)(const DevIndex, const uint8_t*, const uint64_t*, uint64_t, OutT*, uint64_t, int);
    if constexpr (POW2)
        kern = hotf ? k_query_bytes<G, true, OutT, 0, true> : k_query_bytes<G, true, OutT, 0, false>;
    else if (ix.mod_fast_ok)
        kern = hotf ? k_query_bytes<G, false, OutT, 1, true> : k_query_bytes<G, false, OutT, 1, false>;
    else
        kern = hotf ? k_query_bytes<G, false, OutT, 0, true> : k_query_bytes<G, false, OutT, 0, false>;
    constexpr size_t smem = kBytesSmem;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int bps = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, kBytesThreads, smem) != cudaSuccess ||
        bps <= 0)
        bps = 1;
    const uint64_t want = (n + (uint64_t)kBatch * kBytesWarps - 1) / ((uint64_t)kBatch * kBytesWarps);
    const uint64_t cap = (uint64_t)sms * bps;
    const int blocks = (int)(want < cap ? want : cap);
    const cudaError_t e =
        launch_ex_smem(ix, kern, blocks, kBytesThreads, smem, s, ix, d, o, bo, static_cast<OutT*>(out), n,
                       minimal);
    note_launch();
    return e;
}

template <class OutT>
static cudaError_t launch_bw(const DevIndex& ix, int g, bool pow2, const uint8_t* d,
                             const uint64_t* o, uint64_t bo, void* out, uint64_t n, int minimal, cudaStream_t s,
                             int sms) {
#define PH_CASE(G)                                                                 \
    case G:                                                                        \
        return pow2 ? launch_b<G, true, OutT>(ix, d, o, bo, out, n, minimal, s, sms) \
                    : launch_b<G, false, OutT>(ix, d, o, bo, out, n, minimal, s, sms);
    switch (g) {
        PH_CASE(0)
        PH_CASE(1)
        PH_CASE(2)
        PH_CASE(3)
        PH_CASE(4)
    }
#undef PH_CASE
    return cudaErrorInvalidValue;
}

cudaError_t launch_index_bytes_one(const DevIndex& ix, int gamma_kind, bool pow2,
                                   const uint8_t* key, uint32_t len, uint64_t* out, int minimal,
                                   cudaStream_t s) {
    if (len > kOneKeyBytes) return cudaErrorInvalidValue;
    OneKey k{};
    memcpy(k.bytes, key, len);
    k.len = len;
#define PH_CASE(G)                                                                            \
    case G:                                                                                   \
        if (pow2) k_index_bytes_one<G, true><<<1, 32, 0, s>>>(ix, k, out, minimal);          \
        else k_index_bytes_one<G, false><<<1, 32, 0, s>>>(ix, k, out, minimal);              \
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

// T0..T3 once in global memory (DevIndex::aes_tab), filled at index creation.
__global__ void k_fill_aes_tab(uint32_t* tab) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;  // 1024 entries
    if (e < 1024) {
        const uint32_t v = t0_entry(e & 255);
        tab[e] = __funnelshift_l(v, v, 8 * (e >> 8));
    }
}
cudaError_t launch_fill_aes_tab(uint32_t* tab, cudaStream_t s) {
    k_fill_aes_tab<<<4, 256, 0, s>>>(tab);
    return cudaGetLastError();
}

cudaError_t launch_query_bytes(const DevIndex& ix, int gamma_kind, bool pow2,
                               const uint8_t* bytes, const uint64_t* offsets, uint64_t base_off,
                               void* out, int out_width, uint64_t n, int minimal, cudaStream_t s,
                               int sms) {
    if (n == 0) return cudaSuccess;
    if (out_width == 4)
        return launch_bw<uint32_t>(ix, gamma_kind, pow2, bytes, offsets, base_off, out, n, minimal, s, sms);
    return launch_bw<uint64_t>(ix, gamma_kind, pow2, bytes, offsets, base_off, out, n, minimal, s, sms);
}

}  // namespace phg
