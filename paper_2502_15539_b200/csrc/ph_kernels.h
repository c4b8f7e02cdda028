// ph_kernels.h — internal launcher interface between the C ABI (ph_abi.cu)
// and the kernels (ph_query.cu, ph_query_bytes.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "ph_device.cuh"

namespace phg {

// Launch `kernel` with the index's persisting-L2 access-policy window over the hot
// pilot region (a per-launch attribute: the caller's stream is not modified).
template <class... KArgs, class... Args>
inline cudaError_t launch_ex_smem(const DevIndex& ix, void (*kernel)(KArgs...), unsigned grid,
                                  unsigned block, size_t smem, cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    unsigned na = 0;
    if (ix.window_bytes) {
        attr[na].id = cudaLaunchAttributeAccessPolicyWindow;
        attr[na].val.accessPolicyWindow.base_ptr = const_cast<uint8_t*>(ix.pilots);
        attr[na].val.accessPolicyWindow.num_bytes = ix.window_bytes;
        attr[na].val.accessPolicyWindow.hitRatio = ix.window_hit_ratio;
        attr[na].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        attr[na].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        na++;
    }
    cfg.attrs = na ? attr : nullptr;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}
template <class... KArgs, class... Args>
inline cudaError_t launch_ex(const DevIndex& ix, void (*kernel)(KArgs...), unsigned grid,
                             unsigned block, cudaStream_t s, Args... args) {
    return launch_ex_smem(ix, kernel, grid, block, 0, s, args...);
}

// Scratch for the deferred remap (k_remap_patch); idx == nullptr selects the inline
// warp-compacted remap instead. Every warp of the query grid owns a private list of
// cap / (grid warps) entries (no atomics) and writes its count to counts[warp].
struct RemapList {
    uint64_t* idx;
    uint64_t* rem;
    uint32_t* counts;   // >= kMaxRemapLists entries
    uint64_t cap;       // total entries
};
constexpr uint32_t kMaxRemapLists = 1u << 16;

cudaError_t launch_query_u64(const DevIndex& ix, int gamma_kind, bool pow2, const uint64_t* keys,
                             void* out, int out_width, uint64_t n, int minimal, cudaStream_t s,
                             int sms, const RemapList& rl = RemapList{nullptr, nullptr, nullptr, 0});

cudaError_t launch_query_bytes(const DevIndex& ix, int gamma_kind, bool pow2,
                               const uint8_t* bytes, const uint64_t* offsets, uint64_t base_off,
                               void* out, int out_width, uint64_t n, int minimal, cudaStream_t s,
                               int sms);

cudaError_t launch_fill_aes_tab(uint32_t* tab, cudaStream_t s);
// One u64 key as a launch parameter (single-key index()).
cudaError_t launch_index_u64_one(const DevIndex& ix, int gamma_kind, bool pow2, uint64_t key,
                                 uint64_t* out, int minimal, cudaStream_t s);
// One string key of at most 256 bytes, passed in the launch parameters (single-key index()).
cudaError_t launch_index_bytes_one(const DevIndex& ix, int gamma_kind, bool pow2,
                                   const uint8_t* key, uint32_t len, uint64_t* out, int minimal,
                                   cudaStream_t s);

cudaError_t launch_query_kmers(const DevIndex& ix, int gamma_kind, bool pow2, const uint64_t* seq,
                               uint64_t n_bases, int k, void* out, int out_width, int minimal,
                               cudaStream_t s, int sms,
                               const RemapList& rl = RemapList{nullptr, nullptr, nullptr, 0});

// Partitioned path (ph_partition.cu). src_kind 0: keys = u64 keys; 1: keys = packed
// sequence (seq_words, kbits), n = number of windows. scratch >= partition_scratch_bytes.
uint64_t partition_scratch_bytes(uint64_t n, uint32_t G, int out_width);
cudaError_t launch_query_partitioned(const DevIndex& ix, int gamma_kind, bool pow2,
                                     const uint64_t* keys, int src_kind, uint64_t seq_words,
                                     uint32_t kbits, void* out, int out_width, uint64_t n,
                                     int minimal, uint32_t G, void* scratch, cudaStream_t s,
                                     int sms);

// Device-side check violations of a -DPH_CHECKS build (ph_partition.cu); -1 otherwise.
int check_errors(uint64_t* count, uint64_t* line);

// Per-pass event timing of the partitioned path (A, B, C), summed over the timed calls.
void set_pass_timing(bool on);
int pass_times(double* ms_sums, int* calls);

// Construction assist (ph_build.cu): hash + sort + part offsets, synchronous on s.
cudaError_t build_prepare_u64(const uint64_t* keys, uint64_t n, uint64_t P, uint64_t S,
                              uint64_t seed, uint64_t* hashes, uint64_t* offsets, int* status,
                              cudaStream_t s, int sms);

// ph_query_bytes.cu: the string hash of every key as u64 pre-images of the integer hash
// (string-key construction). ix: seed, hash_algo and AES round keys only.
cudaError_t launch_hash_bytes(const DevIndex& ix, const uint8_t* bytes, const uint64_t* offsets,
                              uint64_t* out, uint64_t n, uint64_t cinv, cudaStream_t s, int sms);

// ph_search.cu: the per-part pilot search on the GPU (one CTA per part, 256 pilots at once).
size_t search_smem_bytes(uint64_t S);
int search_check_errors(uint64_t* count, uint64_t* line);  // checked builds (ph_search.cu)
bool search_parts_supported(uint64_t S, uint64_t B, uint64_t max_part);
cudaError_t search_parts_gpu(const uint64_t* d_hashes, const uint64_t* d_off, uint64_t n, uint64_t P,
                             uint64_t S, uint64_t B, uint64_t seed, int fn, const uint64_t* d_opt,
                             uint64_t max_part, uint8_t* d_pilots, uint32_t* d_taken,
                             unsigned long long* h_status, unsigned long long* h_by_pct,
                             cudaStream_t s, int sms);

// Bucket-size histogram of a key set (stats.cpp:59-61): hist_out[s] for s < min(cap, *len).
cudaError_t bucket_size_hist(const DevIndex& ix, int gamma_kind, const uint64_t* keys, uint64_t n,
                             uint64_t* hist_out, uint64_t cap, uint64_t* len_out, cudaStream_t s,
                             int sms);

// Gather-only replay of the pilot reads at the true bucket addresses (bench.py roofline).
cudaError_t launch_gather_replay(const DevIndex& ix, int gamma_kind, const uint64_t* keys,
                                 uint64_t n, uint32_t* sink, cudaStream_t s, int sms);

cudaError_t launch_relayout(const uint8_t* src, uint8_t* dst, uint64_t P, uint64_t B, uint64_t H,
                            cudaStream_t s);
cudaError_t launch_verify(const void* out, int out_width, uint64_t count, uint64_t n,
                          unsigned int* bits, unsigned long long* bad, cudaStream_t s, int sms);

uint64_t launch_count();
void note_launch();
void set_launch(int threads, int bps);
void set_regime(int r);

}  // namespace phg
