/* TEST INFRASTRUCTURE ONLY — plain-C restatement of PtrHash's query path.
 *
 * This is the CPU checker the GPU kernels are compared against in tests/ and
 * the "port" CPU baseline in bench.py. It is never linked into, or called by,
 * the product library (paper_2502_15539_b200/libph_gpu.so).
 *
 * Each function cites the reference file:line it restates (paths relative to
 * /root/reference/proj). Parity of this restatement is pinned two ways:
 *   - against the compiled reference itself (oracle/_ref/libptrhash_ref.so,
 *     built from the reference sources by oracle/Makefile), and
 *   - against the known-answer vectors committed in tests/golden/ (generated
 *     from that reference by tests/golden/gen_golden.py).
 */
#include "ph_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

static const uint64_t kC = 0x517cc1b727220a95ULL;      /* hash.hpp:13 */
static const uint64_t kGolden = 0x9e3779b97f4a7c15ULL; /* common.hpp:60 */
static const uint64_t kP1 = 0x8bb84b93962eacc9ULL;     /* hash.cpp:83-85 */
static const uint64_t kP2 = 0x2d358dccaa6c78a5ULL;
static const uint64_t kP3 = 0x4b33a62ed433d4a3ULL;

/* common.hpp:13-15 */
uint64_t pho_mul_hi(uint64_t a, uint64_t b) { return (uint64_t)(((u128)a * b) >> 64); }

/* common.hpp:54-58 */
uint64_t pho_mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

/* hash.hpp:27 */
uint64_t pho_hash_int(uint64_t key, uint64_t seed) { return kC * (key ^ seed); }
/* hash.hpp:30-32 */
uint64_t pho_hash_pilot(uint64_t pilot, uint64_t seed) { return kC * (pilot ^ seed); }

/* ---- bucket functions, bucket_fn.hpp:18-58 and bucket_fn.cpp:10-56 ---- */

static uint64_t g_opt_table[65537];
static int g_opt_ready = 0;

/* bucket_fn.cpp:16-39: filled with double ln, clamped non-decreasing. */
static void opt_table_init(void) {
    if (g_opt_ready) return;
    const double eps = 1.0 / 256.0;
    const double scale = ldexp(1.0, 64);
    uint64_t prev = 0;
    for (size_t i = 0; i <= 65536; i++) {
        const double x = (double)i / 65536.0;
        double y = x;
        if (x < 1.0) y = x + (1.0 - eps) * (1.0 - x) * log(1.0 - x);
        const double scaled = y * scale;
        uint64_t u;
        if (scaled >= scale) u = UINT64_MAX;
        else if (scaled <= 0.0) u = 0;
        else u = (uint64_t)scaled;
        if (u < prev) u = prev;
        g_opt_table[i] = u;
        prev = u;
    }
    g_opt_ready = 1;
}

const uint64_t* pho_optimal_table(void) {
    opt_table_init();
    return g_opt_table;
}

uint64_t pho_gamma(int kind, uint64_t x) {
    switch (kind) {
        case 0: return x;                      /* linear, :20 */
        case 1: return pho_mul_hi(x, x);       /* quadratic, :22 */
        case 2: {                              /* cubic, :27-32 */
            const uint64_t x2 = pho_mul_hi(x, x);
            const uint64_t x3 = pho_mul_hi(x2, x);
            const uint64_t half = (uint64_t)(((u128)x2 + x3) >> 1);
            return (uint64_t)(((u128)half * 255) >> 8) + (x >> 8);
        }
        case 3: {                              /* skewed, :34-39 */
            const uint64_t sx = (uint64_t)(((u128)3 << 64) / 5);
            const uint64_t sy = (uint64_t)(((u128)3 << 64) / 10);
            if (x < sx) return x >> 1;
            return sy + (uint64_t)(((u128)(x - sx) * 7) >> 2);
        }
        case 4: {                              /* optimal, bucket_fn.cpp:49-56 */
            opt_table_init();
            const uint64_t idx = x >> 48;
            const uint64_t frac = x & ((1ULL << 48) - 1);
            const uint64_t lo = g_opt_table[idx], hi = g_opt_table[idx + 1];
            return lo + (uint64_t)(((u128)(hi - lo) * frac) >> 48);
        }
    }
    return x;
}

/* ---- reduce.hpp:27-77 ---- */
void pho_fastmod_magic(uint64_t S, uint64_t* hi, uint64_t* lo) {
    const u128 m = (~(u128)0) / S + 1;
    *hi = (uint64_t)(m >> 64);
    *lo = (uint64_t)m;
}

static uint64_t fastmod(uint64_t mhi, uint64_t mlo, uint64_t x, uint64_t S) {
    const uint64_t lb_lo = mlo * x;
    const uint64_t lb_hi = mhi * x + pho_mul_hi(mlo, x);
    const u128 t = (u128)lb_hi * S + (((u128)lb_lo * S) >> 64);
    return (uint64_t)(t >> 64);
}

static int is_pow2(uint64_t x) { return x != 0 && (x & (x - 1)) == 0; }

uint64_t pho_reduce(uint64_t S, uint64_t x) {
    if (is_pow2(S)) return pho_mul_hi(kC, x) & (S - 1); /* :68 */
    uint64_t hi, lo;
    pho_fastmod_magic(S, &hi, &lo);
    return fastmod(hi, lo, x, S); /* :69 */
}

/* bucket_fn.hpp:66-72 */
void pho_part_and_bucket(uint64_t h, uint64_t P, uint64_t B, int fn, uint64_t* part,
                         uint64_t* bucket) {
    const u128 prod = (u128)P * h;
    *part = (uint64_t)(prod >> 64);
    *bucket = pho_mul_hi(B, pho_gamma(fn, (uint64_t)prod));
}

/* ---- CacheLineEF decode, cacheline_ef.hpp:38-42, :58-73, :86-90 ----
 * Independent bit-by-bit select (the style of tests/oracles.hpp:40-60). */
static uint64_t le64(const uint8_t* p) {
    uint64_t v = 0;
    for (int i = 7; i >= 0; i--) v = (v << 8) | p[i];
    return v;
}
static uint32_t le32(const uint8_t* p) {
    return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}

uint64_t pho_clef_get(const uint8_t* b, size_t i) {
    const uint64_t off = le32(b);
    const uint64_t m[2] = {le64(b + 4), le64(b + 12)};
    uint32_t rank = (uint32_t)i, pos = 0;
    for (pos = 0; pos < 128; pos++) {
        if ((m[pos >> 6] >> (pos & 63)) & 1) {
            if (rank == 0) break;
            rank--;
        }
    }
    return (off << 8) + ((uint64_t)(pos - i) << 8) + b[20 + i];
}

/* ---- Elias-Fano get, elias_fano.cpp:51-72 ---- */
static uint64_t ef_low_value(const pho_index* ix, uint64_t i) {
    const unsigned l = ix->ef_low_bits;
    if (l == 0) return 0;
    const uint64_t bitpos = i * l;
    uint64_t v = ix->ef_low[bitpos / 64] >> (bitpos % 64);
    if (bitpos % 64 + l > 64) v |= ix->ef_low[bitpos / 64 + 1] << (64 - bitpos % 64);
    return v & ((1ULL << l) - 1);
}

static uint64_t ef_get(const pho_index* ix, uint64_t i) {
    const uint64_t sample = ix->ef_samples[i / 512];
    uint64_t word = sample >> 16;
    uint32_t want = (uint32_t)(sample & 0xffff) + (uint32_t)(i % 512);
    for (;;) {
        const uint32_t c = (uint32_t)__builtin_popcountll(ix->ef_high[word]);
        if (want < c) break;
        want -= c;
        word++;
    }
    uint64_t w = ix->ef_high[word];
    uint32_t bit = 0;
    for (;;) { /* rank-th set bit, naive */
        if (w & 1) {
            if (want == 0) break;
            want--;
        }
        w >>= 1;
        bit++;
    }
    const uint64_t pos = word * 64 + bit;
    return ((pos - i) << ix->ef_low_bits) | ef_low_value(ix, i);
}

/* ---- string hashes, hash.cpp:53-193 ---- */
static uint64_t mum(uint64_t a, uint64_t b) { /* :53-56 */
    const u128 r = (u128)a * b;
    return (uint64_t)r ^ (uint64_t)(r >> 64);
}
static uint64_t rd64(const uint8_t* p) { return le64(p); }
static uint64_t rd32(const uint8_t* p) { return le32(p); }
static uint64_t read_tail(const uint8_t* p, size_t len) { /* :71-81 */
    if (len >= 4) return rd32(p) | (rd32(p + len - 4) << 32);
    return (uint64_t)p[0] | ((uint64_t)p[len >> 1] << 8) | ((uint64_t)p[len - 1] << 16);
}
static uint64_t portable_hash64(const uint8_t* p, size_t len, uint64_t seed) { /* :87-104 */
    uint64_t acc = seed ^ mum((uint64_t)len ^ kP1, seed ^ kP2);
    size_t i = 0;
    while (i + 16 <= len) {
        acc = mum(rd64(p + i) ^ kP1, rd64(p + i + 8) ^ acc);
        i += 16;
    }
    uint64_t a = 0, b = 0;
    if (len - i > 8) {
        a = rd64(p + i);
        b = read_tail(p + i + 8, len - i - 8);
    } else if (len > i) {
        a = read_tail(p + i, len - i);
    }
    acc = mum(a ^ kP2 ^ (uint64_t)len, b ^ acc ^ kP3);
    return mum(acc, acc ^ kP1);
}

/* Software AES round with Intel AESENC/AESENCLAST semantics (what
 * _mm_aesenc_si128 computes in hash.cpp:114-141). State byte i sits at row
 * i%4, column i/4. The S-box is generated from GF(2^8) inverses. */
static uint8_t g_sbox[256];
static int g_sbox_ready = 0;
static uint8_t gf_mul(uint8_t a, uint8_t b) {
    uint8_t r = 0;
    while (b) {
        if (b & 1) r ^= a;
        a = (uint8_t)((a << 1) ^ ((a & 0x80) ? 0x1b : 0));
        b >>= 1;
    }
    return r;
}
static void sbox_init(void) {
    if (g_sbox_ready) return;
    for (int x = 0; x < 256; x++) {
        uint8_t inv = 0;
        if (x) {
            for (int y = 1; y < 256; y++)
                if (gf_mul((uint8_t)x, (uint8_t)y) == 1) { inv = (uint8_t)y; break; }
        }
        uint8_t s = inv;
        for (int r = 1; r <= 4; r++) s ^= (uint8_t)((inv << r) | (inv >> (8 - r)));
        g_sbox[x] = (uint8_t)(s ^ 0x63);
    }
    g_sbox_ready = 1;
}
void pho_aesenc(uint8_t st[16], const uint8_t key[16], int last) {
    sbox_init();
    uint8_t t[16];
    for (int c = 0; c < 4; c++)
        for (int r = 0; r < 4; r++) t[r + 4 * c] = g_sbox[st[r + 4 * ((c + r) & 3)]];
    if (!last) {
        for (int c = 0; c < 4; c++) {
            const uint8_t a0 = t[4 * c], a1 = t[4 * c + 1], a2 = t[4 * c + 2], a3 = t[4 * c + 3];
            t[4 * c + 0] = (uint8_t)(gf_mul(a0, 2) ^ gf_mul(a1, 3) ^ a2 ^ a3);
            t[4 * c + 1] = (uint8_t)(a0 ^ gf_mul(a1, 2) ^ gf_mul(a2, 3) ^ a3);
            t[4 * c + 2] = (uint8_t)(a0 ^ a1 ^ gf_mul(a2, 2) ^ gf_mul(a3, 3));
            t[4 * c + 3] = (uint8_t)(gf_mul(a0, 3) ^ a1 ^ a2 ^ gf_mul(a3, 2));
        }
    }
    for (int i = 0; i < 16; i++) st[i] = t[i] ^ key[i];
}
static void set128(uint8_t out[16], uint64_t hi, uint64_t lo) { /* _mm_set_epi64x(hi, lo) */
    for (int i = 0; i < 8; i++) {
        out[i] = (uint8_t)(lo >> (8 * i));
        out[8 + i] = (uint8_t)(hi >> (8 * i));
    }
}
static void aes_core(const uint8_t* p, size_t len, uint64_t seed, uint64_t* hi, uint64_t* lo) {
    uint8_t k0[16], k1[16], st[16], blk[16];
    set128(k0, seed ^ kP1, seed + kGolden);                                 /* :116-117 */
    set128(k1, pho_mix64(seed) ^ kP2, (~seed) * 0x6c62272e07bb0143ULL);     /* :118-119 */
    set128(st, (uint64_t)len * kC, seed ^ (uint64_t)len);                  /* :120-121 */
    pho_aesenc(st, k0, 0);
    size_t i = 0;
    while (i + 16 <= len) { /* :125-129 */
        for (int j = 0; j < 16; j++) st[j] ^= p[i + j];
        pho_aesenc(st, k1, 0);
        i += 16;
    }
    if (i < len) { /* :130-136 */
        memset(blk, 0, 16);
        memcpy(blk, p + i, len - i);
        blk[15] ^= (uint8_t)(len - i);
        for (int j = 0; j < 16; j++) st[j] ^= blk[j];
        pho_aesenc(st, k1, 0);
    }
    pho_aesenc(st, k0, 0); /* :138-140 */
    pho_aesenc(st, k1, 0);
    pho_aesenc(st, k0, 1);
    *lo = le64(st);
    *hi = le64(st + 8);
}

/* hash.cpp:159-193 */
void pho_hash_bytes(const uint8_t* p, size_t len, uint64_t seed, int algo, uint64_t* hi,
                    uint64_t* lo) {
    switch (algo) {
        case 1: case 2: {
            uint64_t h, l;
            aes_core(p, len, seed, &h, &l);
            if (algo == 1) { /* :148-151 */
                const uint64_t v = h ^ (l * kC);
                *hi = *lo = v;
            } else {
                *hi = h;
                *lo = l;
            }
            return;
        }
        case 4:
            *hi = portable_hash64(p, len, seed ^ kP3);
            *lo = portable_hash64(p, len, pho_mix64(seed) + kGolden);
            return;
        default: { /* 0 (fx64 on bytes) and 3 (portable64) */
            const uint64_t v = portable_hash64(p, len, seed);
            *hi = *lo = v;
            return;
        }
    }
}

/* ---- PTRH v1 parsing, serde.hpp:12-31 / serde.cpp:176-240 ---- */
typedef struct { const uint8_t* p; size_t len, pos; int bad; } rd_t;
static int need(rd_t* r, size_t n) {
    if (r->bad || r->pos + n > r->len) { r->bad = 1; return 0; }
    return 1;
}
static uint8_t r8(rd_t* r) { return need(r, 1) ? r->p[r->pos++] : 0; }
static uint64_t r64(rd_t* r) {
    if (!need(r, 8)) return 0;
    const uint64_t v = le64(r->p + r->pos);
    r->pos += 8;
    return v;
}
static uint64_t* r64_array(rd_t* r, uint64_t max_len, uint64_t* n_out) {
    const uint64_t n = r64(r);
    if (r->bad || n > max_len || !need(r, n * 8)) { r->bad = 1; return NULL; }
    uint64_t* v = (uint64_t*)malloc((n ? n : 1) * 8);
    for (uint64_t i = 0; i < n; i++) v[i] = r64(r);
    *n_out = n;
    return v;
}

int pho_parse(const uint8_t* bytes, size_t len, pho_index* ix, const char** err) {
    memset(ix, 0, sizeof(*ix));
    rd_t r = {bytes, len, 0, 0};
#define FAIL(msg) do { *err = msg; pho_release(ix); return 1; } while (0)
    if (len < 72) FAIL("index file truncated");
    if (memcmp(bytes, "PTRH", 4) != 0) FAIL("not an index file (bad magic)");
    if (le32(bytes + 4) != 1) FAIL("unsupported index format version");
    r.pos = 8;
    ix->key_kind = r8(&r);
    ix->hash_algo = r8(&r);
    ix->bucket_fn = r8(&r);
    ix->remap_kind = r8(&r);
    ix->reduce_kind = r8(&r);
    r.pos += 3;
    if (ix->key_kind > 1) FAIL("unknown key kind id");
    if (ix->hash_algo > 4) FAIL("unknown hash algorithm id");
    if (ix->bucket_fn > 4) FAIL("unknown bucket function id");
    if (ix->remap_kind > 2) FAIL("unknown remap kind id");
    if (ix->reduce_kind > 2) FAIL("unknown reduce kind id");
    ix->n = r64(&r);
    ix->P = r64(&r);
    ix->S = r64(&r);
    ix->B = r64(&r);
    ix->seed = r64(&r);
    const uint64_t pilots_len = r64(&r), remap_len = r64(&r);
    if (ix->n == 0 || ix->P == 0 || ix->S == 0) FAIL("index file: degenerate shape");
    if ((u128)ix->P * ix->S > ((u128)1 << 62) || (u128)ix->P * ix->B > ((u128)1 << 62))
        FAIL("index file: shape out of range");
    if (ix->n > ix->P * ix->S) FAIL("index file: n exceeds the slot count");
    if (pilots_len != ix->P * ix->B) FAIL("index file: pilot length does not match shape");
    if (len - 72 != pilots_len + remap_len) FAIL("index file: payload length mismatch");
    ix->pilots = bytes + 72;
    ix->remap = bytes + 72 + pilots_len;
    ix->remap_len = remap_len;
    const uint64_t count = ix->P * ix->S - ix->n;
    if (ix->remap_kind == 0) {
        if (remap_len != count * 4) FAIL("index file: bad plain remap length");
    } else if (ix->remap_kind == 1) {
        if (remap_len != (count + 43) / 44 * 64) FAIL("index file: bad cacheline-ef remap length");
    } else {
        rd_t e = {ix->remap, remap_len, 0, 0};
        ix->ef_count = r64(&e);
        ix->ef_universe = r64(&e);
        ix->ef_low_bits = r8(&e);
        if (e.bad) FAIL("index file truncated");
        if (ix->ef_count != count) FAIL("index file: bad elias-fano count");
        ix->ef_low = r64_array(&e, remap_len / 8 + 1, &ix->ef_low_n);
        ix->ef_high = r64_array(&e, remap_len / 8 + 1, &ix->ef_high_n);
        ix->ef_samples = r64_array(&e, remap_len / 8 + 1, &ix->ef_samples_n);
        if (e.bad) FAIL("index file: bad elias-fano payload");
        if (e.pos != remap_len) FAIL("index file: trailing bytes");
    }
    ix->pow2 = is_pow2(ix->S);
    if (!ix->pow2) {
        if (ix->S >= (1ULL << 32)) FAIL("reduce: fastmod needs S < 2^32");
        pho_fastmod_magic(ix->S, &ix->magic_hi, &ix->magic_lo);
    }
#undef FAIL
    return 0;
}

void pho_release(pho_index* ix) {
    free(ix->ef_low);
    free(ix->ef_high);
    free(ix->ef_samples);
    ix->ef_low = ix->ef_high = ix->ef_samples = NULL;
}

/* ---- query, index.hpp:91-100 ---- */
uint64_t pho_slot_of(const pho_index* ix, uint64_t hi, uint64_t lo) {
    uint64_t part, bucket;
    pho_part_and_bucket(hi, ix->P, ix->B, ix->bucket_fn, &part, &bucket);
    const uint8_t pilot = ix->pilots[part * ix->B + bucket];
    const uint64_t y = lo ^ pho_hash_pilot(pilot, ix->seed);
    const uint64_t local =
        ix->pow2 ? (pho_mul_hi(kC, y) & (ix->S - 1)) : fastmod(ix->magic_hi, ix->magic_lo, y, ix->S);
    return part * ix->S + local;
}

/* remap.hpp:34-45 */
uint64_t pho_remap_slot(const pho_index* ix, uint64_t slot) {
    if (slot < ix->n) return slot;
    const uint64_t i = slot - ix->n;
    switch (ix->remap_kind) {
        case 0: return le32(ix->remap + 4 * i);
        case 1: return pho_clef_get(ix->remap + 64 * (i / 44), i % 44);
        default: return ef_get(ix, i);
    }
}

uint64_t pho_index_u64(const pho_index* ix, uint64_t key, int minimal) {
    const uint64_t h = pho_hash_int(key, ix->seed);
    const uint64_t slot = pho_slot_of(ix, h, h);
    return minimal ? pho_remap_slot(ix, slot) : slot;
}

uint64_t pho_index_bytes(const pho_index* ix, const uint8_t* p, size_t len, int minimal) {
    uint64_t hi, lo;
    pho_hash_bytes(p, len, ix->seed, ix->hash_algo, &hi, &lo);
    const uint64_t slot = pho_slot_of(ix, hi, lo);
    return minimal ? pho_remap_slot(ix, slot) : slot;
}

void pho_query_u64(const pho_index* ix, const uint64_t* keys, size_t n, uint64_t* out,
                   int minimal) {
    for (size_t i = 0; i < n; i++) out[i] = pho_index_u64(ix, keys[i], minimal);
}

void pho_query_bytes(const pho_index* ix, const uint8_t* data, const uint64_t* offsets, size_t n,
                     uint64_t* out, int minimal) {
    for (size_t i = 0; i < n; i++)
        out[i] = pho_index_bytes(ix, data + offsets[i], offsets[i + 1] - offsets[i], minimal);
}

/* corpus.hpp:14-16 */
uint64_t pho_corpus_u64(uint64_t i, uint64_t gen_seed) {
    return pho_mix64(gen_seed + (i + 1) * kGolden);
}

/* Bulk host generators for the synthetic workloads (bench.py's reference arm). */
void pho_gen_corpus(uint64_t* out, uint64_t start, uint64_t count, uint64_t gen_seed) {
    for (uint64_t i = 0; i < count; i++) out[i] = pho_corpus_u64(start + i, gen_seed);
}
void pho_gen_perm_keys(uint64_t* out, uint64_t start, uint64_t count, uint64_t n,
                       uint64_t gen_seed, uint64_t perm_seed) {
    for (uint64_t i = 0; i < count; i++)
        out[i] = pho_corpus_u64(pho_feistel_perm(start + i, n, perm_seed), gen_seed);
}
void pho_gen_sample_keys(uint64_t* out, uint64_t start, uint64_t count, uint64_t n,
                         uint64_t gen_seed, uint64_t sample_seed) {
    for (uint64_t i = 0; i < count; i++)
        out[i] = pho_corpus_u64(pho_mix64(sample_seed + (start + i + 1) * kGolden) % n, gen_seed);
}

/* Config-4 string corpus: string i has len = 8 + r0 % 57 bytes of printable ASCII
 * 0x21 + mix64(r0 + (t+1)*golden) % 94, with r0 = mix64(seed + (i+1)*golden). Writes the
 * string into out (>= 64 bytes) and returns its length. */
uint32_t pho_gen_string(uint64_t i, uint64_t seed, uint8_t* out) {
    const uint64_t r0 = pho_mix64(seed + (i + 1) * kGolden);
    const uint32_t len = 8 + (uint32_t)(r0 % 57);
    for (uint32_t t = 0; t < len; t++) out[t] = (uint8_t)(0x21 + pho_mix64(r0 + (t + 1) * kGolden) % 94);
    return len;
}
/* Strings src(start..start+count) concatenated into data at data_off, offsets[] relative to
 * data_off's base (offsets[c] is written for c in [0, count]); src = perm(i) if perm_seed != 0. */
uint64_t pho_gen_strings(uint64_t start, uint64_t count, uint64_t n, uint64_t seed,
                         uint64_t perm_seed, uint8_t* data, uint64_t* offsets, uint64_t base) {
    uint64_t pos = base;
    for (uint64_t c = 0; c < count; c++) {
        const uint64_t i = start + c;
        const uint64_t src = perm_seed ? pho_feistel_perm(i, n, perm_seed) : i;
        offsets[c] = pos;
        pos += pho_gen_string(src, seed, data + pos);
    }
    offsets[count] = pos;
    return pos;
}

/* k-mer workload (BASELINE.json config 5; the GPU's fused front end is checked against
 * this): sequence word w = mix64(seed + (w+1)*golden), bases 2-bit MSB-first (A=0 C=1 G=2
 * T=3); key i = bases i..i+k-1 with the first base in the most significant bits. */
void pho_gen_dna(uint64_t* out, uint64_t start_word, uint64_t nwords, uint64_t seed) {
    for (uint64_t w = 0; w < nwords; w++) out[w] = pho_mix64(seed + (start_word + w + 1) * kGolden);
}
void pho_kmers(const uint64_t* seq, uint64_t n_bases, int k, uint64_t start, uint64_t count,
               uint64_t* out) {
    for (uint64_t c = 0; c < count; c++) {
        const uint64_t i = start + c;
        uint64_t key = 0;
        for (int t = 0; t < k; t++) { /* base by base, no word tricks */
            const uint64_t j = i + (uint64_t)t;
            const uint64_t b = (seq[j / 32] >> (2 * (31 - j % 32))) & 3;
            key = (key << 2) | b;
        }
        (void)n_bases;
        out[c] = key;
    }
}

/* Seeded permutation of [0,n) used as the "shuffled query order" of the
 * synthetic workloads (ours, not the reference's): a 4-round balanced Feistel
 * network over the smallest even-bit domain >= n, with cycle walking. The GPU
 * harness computes the identical function. */
uint64_t pho_feistel_perm(uint64_t i, uint64_t n, uint64_t seed) {
    unsigned bits = 2;
    while (bits < 64 && (1ULL << bits) < n) bits += 2;
    const unsigned h = bits / 2;
    const uint64_t mask = (1ULL << h) - 1;
    uint64_t x = i;
    do {
        uint64_t L = x >> h, R = x & mask;
        for (uint64_t r = 0; r < 4; r++) {
            const uint64_t t = L ^ (pho_mix64(R ^ (seed + (r + 1) * kGolden)) & mask);
            L = R;
            R = t;
        }
        x = (L << h) | R;
    } while (x >= n);
    return x;
}
