/* TEST INFRASTRUCTURE ONLY — plain-C restatement of the PtrHash query path
 * (reference: /root/reference/proj, C++). Used by tests/ and bench.py's
 * cpu_baseline leg as a checker; never linked into the product library.
 * Pinned against the compiled reference (oracle/_ref/libptrhash_ref.so) and
 * the golden vectors in tests/golden/ (see tests/test_oracle.py). */
#ifndef PH_ORACLE_H
#define PH_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- primitives ---- */
uint64_t pho_mul_hi(uint64_t a, uint64_t b);
uint64_t pho_mix64(uint64_t z);
uint64_t pho_hash_int(uint64_t key, uint64_t seed);
uint64_t pho_hash_pilot(uint64_t pilot, uint64_t seed);
uint64_t pho_gamma(int kind, uint64_t x);
const uint64_t* pho_optimal_table(void); /* 65537 entries, bucket_fn.cpp:13-40 */
void pho_fastmod_magic(uint64_t S, uint64_t* hi, uint64_t* lo);
uint64_t pho_reduce(uint64_t S, uint64_t x);
void pho_part_and_bucket(uint64_t h, uint64_t P, uint64_t B, int fn, uint64_t* part,
                         uint64_t* bucket);
uint64_t pho_clef_get(const uint8_t* block64, size_t i);
void pho_hash_bytes(const uint8_t* p, size_t len, uint64_t seed, int algo, uint64_t* hi,
                    uint64_t* lo);
void pho_aesenc(uint8_t state[16], const uint8_t key[16], int last);

/* ---- index (parsed PTRH v1 bytes; pointers alias the caller's buffer) ---- */
typedef struct pho_index {
    uint8_t key_kind, hash_algo, bucket_fn, remap_kind, reduce_kind;
    uint64_t n, P, S, B, seed;
    const uint8_t* pilots;
    const uint8_t* remap; /* raw payload */
    uint64_t remap_len;
    /* Elias-Fano pieces (copied, aligned) */
    uint64_t ef_count, ef_universe;
    uint8_t ef_low_bits;
    uint64_t *ef_low, *ef_high, *ef_samples;
    uint64_t ef_low_n, ef_high_n, ef_samples_n;
    uint64_t magic_hi, magic_lo;
    int pow2;
} pho_index;

/* Returns 0 on success, nonzero + message on malformed input (serde.cpp:176-240). */
int pho_parse(const uint8_t* bytes, size_t len, pho_index* out, const char** err);
void pho_release(pho_index* ix);

uint64_t pho_slot_of(const pho_index* ix, uint64_t hi, uint64_t lo);
uint64_t pho_remap_slot(const pho_index* ix, uint64_t slot);
uint64_t pho_index_u64(const pho_index* ix, uint64_t key, int minimal);
uint64_t pho_index_bytes(const pho_index* ix, const uint8_t* p, size_t len, int minimal);
void pho_query_u64(const pho_index* ix, const uint64_t* keys, size_t n, uint64_t* out,
                   int minimal);
void pho_query_bytes(const pho_index* ix, const uint8_t* data, const uint64_t* offsets, size_t n,
                     uint64_t* out, int minimal);

/* ---- synthetic workloads shared with the GPU harness ---- */
uint64_t pho_corpus_u64(uint64_t i, uint64_t gen_seed);
uint64_t pho_feistel_perm(uint64_t i, uint64_t n, uint64_t seed);
void pho_gen_corpus(uint64_t* out, uint64_t start, uint64_t count, uint64_t gen_seed);
void pho_gen_perm_keys(uint64_t* out, uint64_t start, uint64_t count, uint64_t n,
                       uint64_t gen_seed, uint64_t perm_seed);
void pho_gen_sample_keys(uint64_t* out, uint64_t start, uint64_t count, uint64_t n,
                         uint64_t gen_seed, uint64_t sample_seed);
void pho_gen_dna(uint64_t* out, uint64_t start_word, uint64_t nwords, uint64_t seed);
uint32_t pho_gen_string(uint64_t i, uint64_t seed, uint8_t* out);
uint64_t pho_gen_strings(uint64_t start, uint64_t count, uint64_t n, uint64_t seed,
                         uint64_t perm_seed, uint8_t* data, uint64_t* offsets, uint64_t base);
void pho_kmers(const uint64_t* seq, uint64_t n_bases, int k, uint64_t start, uint64_t count,
               uint64_t* out);

#ifdef __cplusplus
}
#endif
#endif
