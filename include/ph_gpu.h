/* ph_gpu.h — C ABI of the B200 (sm_100a) PtrHash query path.
 *
 * Drop-in boundary for the reference's query API, PtrHashIndex
 * (/root/reference/proj/include/ptrhash/index.hpp:58-81). The index is the
 * reference's own serialized PTRH v1 file (proj/include/ptrhash/serde.hpp:12-31),
 * uploaded unchanged to one GPU; every query returns exactly the reference's value.
 *
 * Conventions:
 *  - integer status, PH_OK == 0; no exceptions cross the ABI; message via
 *    ph_gpu_last_error() (thread-local);
 *  - a ph_gpu_index is immutable after create and safe to use from any number of
 *    host threads and CUDA streams at once (index.hpp:26-31);
 *  - device-pointer entry points are asynchronous on the given stream
 *    (a cudaStream_t passed as void*; NULL = legacy default stream);
 *  - host-pointer entry points are synchronous, like the reference's methods;
 *  - queries have no error path for non-member keys: they return an arbitrary
 *    value below n (minimal) or below P*S (non-minimal), as index.hpp:26-31.
 */
#ifndef PH_GPU_H
#define PH_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ph_gpu_index ph_gpu_index; /* opaque, immutable after create */
typedef void* ph_gpu_stream_t;            /* cudaStream_t */

enum ph_gpu_status {
    PH_OK = 0,
    PH_E_INVALID = 1,  /* bad argument (null pointer, bad width, ...) */
    PH_E_FORMAT = 2,   /* malformed PTRH bytes; same checks as serde.cpp:176-240 */
    PH_E_CUDA = 3,     /* CUDA runtime error (no device, launch failure, ...) */
    PH_E_KEYKIND = 4,  /* u64 query on a string index or vice versa (index.hpp:18-21) */
    PH_E_NOMEM = 5,    /* device or pinned-host allocation failed */
    PH_E_UNSUPPORTED = 6, /* shape outside what the GPU path supports */
    PH_E_DUPLICATE = 7,   /* build: duplicate keys (BuildError::kDuplicateKeys, build.hpp:48-61) */
    PH_E_BUILD_FAILED = 8 /* build: every seed attempt failed (BuildError::kFailed) */
};

/* Output element width for bulk queries: u32 (all configs, n <= 2^32) or u64
 * (the reference's `uint64_t* out`, index.hpp:72-81). */
enum { PH_OUT_U32 = 4, PH_OUT_U64 = 8 };

typedef struct ph_gpu_info {
    uint64_t n;                /* keys (Shape::n, shape.hpp:65-75) */
    uint64_t parts;            /* P */
    uint64_t slots_per_part;   /* S */
    uint64_t buckets_per_part; /* B */
    uint64_t seed;
    uint64_t pilot_bytes;      /* P*B */
    uint64_t remap_values;     /* P*S - n */
    uint64_t remap_bytes;      /* payload bytes resident on the device */
    uint8_t key_kind;          /* 0 u64, 1 bytes (index.hpp:18-21) */
    uint8_t hash_algo;         /* hash.hpp:37-43 */
    uint8_t bucket_fn;         /* shape.hpp:23-29 */
    uint8_t remap_kind;        /* shape.hpp:31-35 */
    uint8_t reduce_kind;       /* header id (reduce.hpp:11-20); informational */
    uint8_t pow2;              /* reduce path actually used: is_power_of_two(S), reduce.hpp:51 */
    int32_t device;
} ph_gpu_info;

/* Parse + validate PTRH v1 bytes (serde.cpp:176-240) and upload pilots and the
 * remap payload to `device`. Replaces deserialize()/load_index() + the
 * PtrHashIndex ctor (serde.cpp:176-260, index.hpp:36-46). */
int ph_gpu_index_create(const uint8_t* ptrh, size_t len, int device, ph_gpu_index** out);
/* load_index (serde.cpp:251-260): mmap + pinned upload of a PTRH v1 file, then exactly
 * ph_gpu_index_create. */
int ph_gpu_index_load(const char* path, int device, ph_gpu_index** out);
int ph_gpu_index_destroy(ph_gpu_index* index);
/* Returns the index's cached per-call scratch (the partitioned path keeps ~29 B/key of its
 * largest batch in the index's memory pool between calls) to the device. Memory still in use
 * by queries in flight is kept; later queries allocate again. */
int ph_gpu_index_trim(const ph_gpu_index* index);
/* Ceiling on the per-call scratch an index keeps cached between calls (the pool's release
 * threshold; default: a quarter of the device's memory). Scratch above it returns to the
 * device at the caller's next synchronisation, so a later large call maps it again (~1 ms
 * per GB). 0 keeps nothing. */
int ph_gpu_index_set_scratch_limit(ph_gpu_index* index, uint64_t bytes);
int ph_gpu_index_info(const ph_gpu_index* index, ph_gpu_info* out);
const char* ph_gpu_last_error(void);

/* ---- device-resident bulk queries (asynchronous on `stream`) ----
 * Replace PtrHashIndex::index_loop / index_batched / index_stream
 * (index.hpp:72-81, index.cpp:15-137): out[i] = minimal ? index(keys[i])
 * : index_no_remap(keys[i]). d_out holds n elements of `out_width` bytes. */
int ph_gpu_query_u64(const ph_gpu_index* index, const uint64_t* d_keys, size_t n, void* d_out,
                     int out_width, int minimal, ph_gpu_stream_t stream);

/* String keys as one concatenated byte buffer + offsets[n+1] (key i is
 * bytes[offsets[i] .. offsets[i+1])). Replaces the span<const std::string>
 * overloads (index.hpp:77-81) with hash_bytes (hash.cpp:159-193). */
int ph_gpu_query_bytes(const ph_gpu_index* index, const uint8_t* d_bytes,
                       const uint64_t* d_offsets, size_t n, void* d_out, int out_width,
                       int minimal, ph_gpu_stream_t stream);

/* k-mer keys, fused (the SSHash use case): the queries are
 * the n_bases-k+1 consecutive k-mers (1 <= k <= 32) of a 2-bit packed DNA sequence, in
 * sequence order. Packing: A=0, C=1, G=2, T=3; word w holds bases 32w..32w+31, base 32w+t
 * at bits 2(31-t) (MSB-first); the key of window i is its k bases with the first base in
 * the most significant bits — the u64 key a caller would otherwise materialise and pass
 * to ph_gpu_query_u64 (identical outputs). d_seq holds ceil(n_bases/32) words. */
int ph_gpu_query_kmers(const ph_gpu_index* index, const uint64_t* d_seq, uint64_t n_bases, int k,
                       void* d_out, int out_width, int minimal, ph_gpu_stream_t stream);

/* ---- host-resident bulk queries (synchronous; the reference's own signature
 * shape: host keys in, host `out` fully overwritten) ----
 * Pipelined H2D -> kernel -> D2H over chunks on several streams. Pinned host
 * buffers are used directly; pageable ones are staged through pinned bounce
 * buffers. */
int ph_gpu_index_stream_u64(const ph_gpu_index* index, const uint64_t* h_keys, size_t n,
                            void* h_out, int out_width, int minimal);
int ph_gpu_index_stream_bytes(const ph_gpu_index* index, const uint8_t* h_bytes,
                              const uint64_t* h_offsets, size_t n, void* h_out, int out_width,
                              int minimal);
/* k-mers of a host-resident packed sequence (layout as ph_gpu_query_kmers); h_out gets
 * n_bases-k+1 elements. */
int ph_gpu_index_stream_kmers(const ph_gpu_index* index, const uint64_t* h_seq, uint64_t n_bases,
                              int k, void* h_out, int out_width, int minimal);

/* ---- single-key queries (synchronous): index() / index_no_remap(),
 * index.hpp:60-64 ---- */
int ph_gpu_index_u64(const ph_gpu_index* index, uint64_t key, int minimal, uint64_t* out);
int ph_gpu_index_bytes(const ph_gpu_index* index, const uint8_t* key, size_t len, int minimal,
                       uint64_t* out);

/* ---- construction assist (not the query path) ---- */
/* The data-parallel phases of one u64 build attempt (construction.cpp:28-60): hash_all
 * (construction.cpp:98-111), scatter_to_parts (engine.hpp:412-474) and each part's
 * std::sort + duplicate check (engine.hpp:505-518), on `device`, synchronous. d_hashes[n]
 * receives the hashes C*(key^seed) in part-major order with every part sorted (the array the
 * reference's pilot search consumes), d_offsets[parts+1] the part boundaries. *status: 0 ok,
 * 1 = a part holds more than slots_per_part keys (the reference's kOversubscribed), 2 = equal
 * hashes (kDuplicateHashes). Its ~9 B/key of device scratch stays cached in a per-device
 * memory pool for later calls. */
int ph_gpu_build_prepare_u64(const uint64_t* d_keys, size_t n, uint64_t parts,
                             uint64_t slots_per_part, uint64_t seed, int device,
                             uint64_t* d_hashes, uint64_t* d_offsets, int* status);

/* ---- construction: the reference's u64 build with its front on the GPU ---- */
/* BuildParams (shape.hpp:46-56). parts/slots_per_part/buckets_per_part all 0: compute_shape
 * (shape.cpp:99-145); all set: build_with_shape (construction.cpp:145-152). */
typedef struct ph_build_params {
    uint32_t alpha_num, alpha_den;   /* load factor in (0, 1] */
    uint32_t lambda_num, lambda_den; /* expected bucket size, >= 1 */
    uint8_t bucket_fn;               /* shape.hpp:23-29 */
    uint8_t remap_kind;              /* shape.hpp:31-35 */
    uint8_t reduce_kind;             /* reduce.hpp:11-20 */
    uint8_t reserved;
    uint32_t max_seed_retries;
    uint64_t seed;
    uint64_t parts, slots_per_part, buckets_per_part;
} ph_build_params;

/* BuildStats (build.hpp:10-45) plus the wall time of each stage. */
typedef struct ph_build_stats {
    uint64_t n, parts, slots_per_part, buckets_per_part;
    uint64_t seed;                       /* of the successful attempt */
    uint32_t attempts;
    uint8_t remap_kind;                  /* actual, after any CacheLineEF fallback */
    uint8_t remap_fell_back;
    uint8_t reserved[2];
    uint64_t total_evictions;
    uint64_t evictions_by_percentile[100];
    uint64_t pilot_bytes, remap_payload_bytes;
    double upload_ms;   /* host keys -> device */
    double prepare_ms;  /* GPU: hash + sort + part offsets, all attempts */
    double search_ms;   /* pilot search over all parts (GPU kernel + copy back, or host threads) */
    double remap_ms;    /* remap table + serialization */
    double total_ms;
} ph_build_stats;

/* preset() (shape.cpp:65-84): "fast", "default", "compact". */
int ph_build_preset(const char* name, ph_build_params* out);
/* compute_shape (shape.cpp:99-145). */
int ph_build_compute_shape(uint64_t n, const ph_build_params* params, uint64_t* parts,
                           uint64_t* slots_per_part, uint64_t* buckets_per_part);
/* build(span<const uint64_t>, params, threads, stats) + serialize() (construction.cpp:139-143,
 * serde.cpp:142-170): the PTRH v1 bytes of the index over the distinct keys keys[0..n), which
 * may be host or device memory. Each attempt hashes and sorts on `device`
 * (ph_gpu_build_prepare_u64) and runs the per-part pilot search there too (one CTA per part,
 * csrc/ph_search.cu; ph_gpu_set_build_search), or on `threads` host threads (0 = all) fed part
 * by part from the device. The bytes equal the reference's for the same keys and parameters. *ptrh is malloc'ed: release it with ph_free. Errors: PH_E_INVALID
 * (bad parameters or shape, empty key set), PH_E_DUPLICATE, PH_E_BUILD_FAILED, PH_E_CUDA,
 * PH_E_NOMEM. */
int ph_gpu_build_u64(const uint64_t* keys, size_t n, const ph_build_params* params,
                     unsigned threads, int device, uint8_t** ptrh, size_t* len,
                     ph_build_stats* stats);
/* build(std::span<const std::string>, params, threads, stats) + serialize()
 * (construction.cpp:154-226) for keys given as concatenated bytes + offsets[n+1] (both host or
 * both device): every key is hashed on `device` with the index's string hash (hash_algo: 1 =
 * aes64, what the reference picks on an x86 host with AES-NI for n < 2^32, hash.cpp:40-46; 3 =
 * portable64), and the 64-bit hashes go through the same sort and pilot search as a u64 build.
 * The bytes equal the reference's build for the same keys, parameters and hash. Equal
 * fingerprints (status of the sort) reseed once, as the reference does; a second time the
 * reference widens to its 128-bit hash, which this builder does not produce: PH_E_UNSUPPORTED
 * (so is n >= 2^32). Other errors as ph_gpu_build_u64. */
int ph_gpu_build_bytes(const uint8_t* bytes, const uint64_t* offsets, size_t n,
                       const ph_build_params* params, int hash_algo, unsigned threads, int device,
                       uint8_t** ptrh, size_t* len, ph_build_stats* stats);
/* Where ph_gpu_build_u64 / ph_gpu_build_bytes run the per-part pilot search (engine.hpp:105-292): 0 (default) on
 * the GPU, one CTA per part (csrc/ph_search.cu), falling back to host threads for shapes the
 * kernel does not take (slots_per_part beyond the shared-memory bitmap, a bucket over 64
 * keys); 1 always on host threads; 2 on the GPU or PH_E_UNSUPPORTED. Either way the bytes are
 * the reference's; ph_build_stats.reserved[0] = 1 reports a GPU search. */
int ph_gpu_set_build_search(int mode);
/* The host stage of one attempt under `seed` (no GPU): hashes[0..n) are the attempt's sorted
 * hashes in part-major order and offsets[parts+1] the part boundaries (what
 * ph_gpu_build_prepare_u64 returns). PH_E_BUILD_FAILED if a part cannot be placed. */
int ph_build_from_sorted_u64(const uint64_t* hashes, const uint64_t* offsets, size_t n,
                             const ph_build_params* params, uint64_t seed, unsigned threads,
                             uint8_t** ptrh, size_t* len, ph_build_stats* stats);
void ph_free(void* p);

/* Build statistics (stats.cpp:59-61; recorded by group_buckets, engine.hpp:304-322) on the
 * index's device, synchronous: hist[s] = number of the P*B buckets holding s of the u64 keys
 * d_keys[0..n) (the key set the index was built from gives the reference's
 * bucket_size_counts). *len = largest size + 1; min(cap, *len) entries are written.
 * PH_E_UNSUPPORTED if a bucket holds more than 2^24 keys. */
int ph_gpu_bucket_sizes(const ph_gpu_index* index, const uint64_t* d_keys, size_t n,
                        uint64_t* hist, size_t cap, size_t* len);

/* ---- verification ---- */
/* verify_bijection (proj/tools/ptrhash.cpp:186-210) on `device`, synchronous: counts the
 * outputs >= n and the repeated outputs among d_out[0..count) (u32 or u64). */
int ph_gpu_verify_bijection(const void* d_out, size_t count, int out_width, uint64_t n,
                            int device, uint64_t* out_of_range, uint64_t* duplicates);

/* Measurement (bench.py's replay bound): the query path's pilot reads alone at
 * the index's true bucket addresses, in the order of d_keys (u64 keys, async on stream):
 * the keys are streamed and each key's pilot byte is gathered as the query kernels do, with
 * no slot arithmetic, remap or output. */
int ph_gpu_gather_replay_u64(const ph_gpu_index* index, const uint64_t* d_keys, size_t n,
                             ph_gpu_stream_t stream);

/* Checked builds only (-DPH_CHECKS; tools/checked_run.py): device-side bounds violations of
 * the partitioned path's staging, bulk copies and scatters plus scratch canary damage, since
 * the last call. PH_E_UNSUPPORTED in normal builds. */
int ph_gpu_check_errors(uint64_t* count, uint64_t* first_line);

/* ---- introspection ---- */
/* Number of query-kernel launches this process made through this library. */
uint64_t ph_gpu_launch_count(void);
/* Minimal queries of at least min_keys keys (default 2^20) defer the slot >= n remap to a
 * second kernel (warp-private lists + k_remap_patch); smaller ones remap inline.
 * UINT64_MAX disables deferral. Results are identical either way. */
int ph_gpu_set_defer_min(uint64_t min_keys);
/* Partitioned path for device-resident u64 / k-mer batches: keys are
 * binned by hash group so each group's pilot slice stays L2-resident, answered, then
 * restored to input order. Needs the file-order pilot layout without a persisting window
 * (the default for pilot arrays > 64 MiB) and ~30 B/key of stream-ordered scratch from the
 * index's pool (falls back to the direct kernel if it cannot be had).
 * 0 = automatic (DRAM-sized pilot arrays, batches >= pilot_bytes/32 keys), 1 = never,
 * 2 = whenever the layout allows. Results are identical. */
int ph_gpu_set_partition(int mode);
/* Profiling aid (one host thread): when on, partitioned-path calls record CUDA events around
 * their three passes (bin, query, unbin; up to 256 calls). ph_gpu_pass_times waits for the
 * recorded calls and returns the summed milliseconds of each pass and the call count;
 * ph_gpu_set_pass_timing resets the record. */
int ph_gpu_set_pass_timing(int on);
int ph_gpu_pass_times(double* ms_sums3, int* calls);
/* Kernel tuning for u64/k-mer queries: 0 = automatic (by pilot bytes vs L2), 1 = the
 * L2-resident tuning, 2 = the DRAM-bound tuning. Tuning/bench knob. */
int ph_gpu_set_regime(int regime);
/* Override the bulk-kernel launch shape (0 = automatic). For tuning/bench. */
int ph_gpu_set_launch(int threads_per_block, int blocks_per_sm);
/* Pilot layout and L2 policy. Default: pilot arrays of at most 64 MiB keep the file order
 * under a persisting L2 window over all of it (hot_bytes = 64 MiB, flags = 0); larger ones
 * keep the file order without a window (hot_bytes = 0, flags = 2), so large batches take the
 * partitioned path. Pilot arrays larger than a nonzero hot_bytes are laid out hot-first: the
 * first hot_bytes/P buckets of every part form a contiguous region covered by a persisting
 * L2 access-policy window (this sets the context's cudaLimitPersistingL2CacheSize).
 * hot_bytes = 0 or flag 2 (no window) keeps the file order and releases the device-wide
 * persisting set-aside (the partitioned path needs both). flag 1: cold-region loads use
 * L2::evict_first. Results are unaffected. Do not call while queries on `index` are in
 * flight. */
int ph_gpu_index_set_l2_policy(ph_gpu_index* index, uint64_t hot_bytes, int flags);

#ifdef __cplusplus
}
#endif
#endif /* PH_GPU_H */
