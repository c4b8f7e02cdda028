// ph_gpu/index.hpp — C++ wrapper over the C ABI (ph_gpu.h) that mirrors the
// reference's query API, ptrhash::PtrHashIndex
// (/root/reference/proj/include/ptrhash/index.hpp:33-115):
//
//   uint64_t index(uint64_t) / index(std::string_view)                 index.hpp:63-64
//   uint64_t index_no_remap(uint64_t) / index_no_remap(std::string_view) index.hpp:60-61
//   void index_loop / index_batched / index_stream(span keys, ..., uint64_t* out, bool minimal)
//                                                                       index.hpp:72-81
// and, for u64 keys, ph_gpu::build(keys, params) for build() + serialize()
// (construction.cpp:113-143): the same PTRH bytes, built on the GPU.
//
// Host spans are staged through the library's pipelined H2D -> kernel -> D2H
// path; the call returns when `out` is complete, like the reference. The
// lookahead / batch_size arguments are accepted for signature parity and do
// not change results (all modes give identical outputs, index.hpp:66-70).
// Errors the reference reports by exception at load time (SerdeError,
// serde.hpp:39-42) are thrown here as ph_gpu::Error; queries never fail for
// non-member keys.
#pragma once

#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "ph_gpu.h"

namespace ph_gpu {

class Error : public std::runtime_error {
  public:
    Error(int code, const std::string& what) : std::runtime_error(what), code_(code) {}
    int code() const { return code_; }

  private:
    int code_;
};

inline void check(int rc) {
    if (rc != PH_OK) throw Error(rc, ph_gpu_last_error());
}

class PtrHashIndex {
  public:
    // From serialized PTRH v1 bytes (what ptrhash::serialize / save_index produce).
    explicit PtrHashIndex(std::span<const uint8_t> ptrh, int device = 0) {
        check(ph_gpu_index_create(ptrh.data(), ptrh.size(), device, &h_));
        check(ph_gpu_index_info(h_, &info_));
    }
    // load_index (serde.cpp:251-260): straight from a PTRH v1 file (mmap + pinned upload).
    static PtrHashIndex load(const char* path, int device = 0) {
        PtrHashIndex ix;
        check(ph_gpu_index_load(path, device, &ix.h_));
        check(ph_gpu_index_info(ix.h_, &ix.info_));
        return ix;
    }
    PtrHashIndex(const PtrHashIndex&) = delete;
    PtrHashIndex& operator=(const PtrHashIndex&) = delete;
    PtrHashIndex(PtrHashIndex&& o) noexcept : h_(o.h_), info_(o.info_) { o.h_ = nullptr; }
    ~PtrHashIndex() {
        if (h_) ph_gpu_index_destroy(h_);
    }

    uint64_t n() const { return info_.n; }
    uint64_t seed() const { return info_.seed; }
    const ph_gpu_info& info() const { return info_; }
    const ph_gpu_index* handle() const { return h_; }

    // ---- single-key queries ----
    uint64_t index_no_remap(uint64_t key) const { return single(key, false); }
    uint64_t index_no_remap(std::string_view key) const { return single(key, false); }
    uint64_t index(uint64_t key) const { return single(key, true); }
    uint64_t index(std::string_view key) const { return single(key, true); }

    // ---- sequence queries over host memory ----
    void index_loop(std::span<const uint64_t> keys, uint64_t* out, bool minimal = true) const {
        check(ph_gpu_index_stream_u64(h_, keys.data(), keys.size(), out, PH_OUT_U64, minimal));
    }
    void index_batched(std::span<const uint64_t> keys, size_t /*batch_size*/, uint64_t* out,
                       bool minimal = true) const {
        index_loop(keys, out, minimal);
    }
    void index_stream(std::span<const uint64_t> keys, size_t /*lookahead*/, uint64_t* out,
                      bool minimal = true) const {
        index_loop(keys, out, minimal);
    }

    void index_loop(std::span<const std::string> keys, uint64_t* out, bool minimal = true) const {
        std::vector<uint8_t> bytes;
        std::vector<uint64_t> offsets;
        concat(keys, bytes, offsets);
        check(ph_gpu_index_stream_bytes(h_, bytes.data(), offsets.data(), keys.size(), out,
                                        PH_OUT_U64, minimal));
    }
    void index_batched(std::span<const std::string> keys, size_t, uint64_t* out,
                       bool minimal = true) const {
        index_loop(keys, out, minimal);
    }
    void index_stream(std::span<const std::string> keys, size_t, uint64_t* out,
                      bool minimal = true) const {
        index_loop(keys, out, minimal);
    }

    // ---- B200-native extras: u32 outputs, concatenated strings, device spans ----
    void index_u32(std::span<const uint64_t> keys, uint32_t* out, bool minimal = true) const {
        check(ph_gpu_index_stream_u64(h_, keys.data(), keys.size(), out, PH_OUT_U32, minimal));
    }
    void index_bytes(const uint8_t* bytes, const uint64_t* offsets, size_t n, uint64_t* out,
                     bool minimal = true) const {
        check(ph_gpu_index_stream_bytes(h_, bytes, offsets, n, out, PH_OUT_U64, minimal));
    }
    // k-mers of a host 2-bit packed sequence (ph_gpu.h layout), in sequence order
    void index_kmers(const uint64_t* seq, uint64_t n_bases, int k, uint32_t* out,
                     bool minimal = true) const {
        check(ph_gpu_index_stream_kmers(h_, seq, n_bases, k, out, PH_OUT_U32, minimal));
    }
    // device-resident, asynchronous on `stream`
    void query_device(const uint64_t* d_keys, size_t n, void* d_out, int out_width, bool minimal,
                      ph_gpu_stream_t stream = nullptr) const {
        check(ph_gpu_query_u64(h_, d_keys, n, d_out, out_width, minimal, stream));
    }
    // returns the cached per-call scratch of large (partitioned) batches to the device
    void trim() const { check(ph_gpu_index_trim(h_)); }

  private:
    uint64_t single(uint64_t key, bool minimal) const {
        uint64_t v = 0;
        check(ph_gpu_index_u64(h_, key, minimal, &v));
        return v;
    }
    uint64_t single(std::string_view key, bool minimal) const {
        uint64_t v = 0;
        check(ph_gpu_index_bytes(h_, reinterpret_cast<const uint8_t*>(key.data()), key.size(),
                                 minimal, &v));
        return v;
    }
    static void concat(std::span<const std::string> keys, std::vector<uint8_t>& bytes,
                       std::vector<uint64_t>& offsets) {
        offsets.resize(keys.size() + 1);
        size_t total = 0;
        for (size_t i = 0; i < keys.size(); i++) {
            offsets[i] = total;
            total += keys[i].size();
        }
        offsets[keys.size()] = total;
        bytes.resize(total ? total : 1);
        for (size_t i = 0; i < keys.size(); i++)
            std::copy(keys[i].begin(), keys[i].end(), bytes.begin() + offsets[i]);
    }

    PtrHashIndex() = default;
    ph_gpu_index* h_ = nullptr;
    ph_gpu_info info_{};
};

// ---- construction (u64 keys) ------------------------------------------------------------
// preset() (shape.cpp:65-84): "fast", "default" or "compact".
inline ph_build_params preset(const char* name) {
    ph_build_params p{};
    check(ph_build_preset(name, &p));
    return p;
}

// build(std::span<const uint64_t>, params, threads, stats) + serialize()
// (/root/reference/proj/src/construction.cpp:113-143, src/serde.cpp:142-174): the PTRH v1
// bytes of the index over the distinct keys, the same bytes the reference produces. Hashing,
// sorting and the per-part pilot search run on `device`; `keys` may be host or device memory.
// Throws Error with PH_E_DUPLICATE (BuildError kDuplicateKeys), PH_E_BUILD_FAILED (kFailed)
// or PH_E_INVALID (kInvalid), build.hpp:48-60.
inline std::vector<uint8_t> build(std::span<const uint64_t> keys, const ph_build_params& params,
                                  unsigned threads = 0, int device = 0,
                                  ph_build_stats* stats = nullptr) {
    uint8_t* bytes = nullptr;
    size_t len = 0;
    check(ph_gpu_build_u64(keys.data(), keys.size(), &params, threads, device, &bytes, &len, stats));
    std::vector<uint8_t> out(bytes, bytes + len);
    ph_free(bytes);
    return out;
}

// build(std::span<const std::string>, params, threads, stats) + serialize()
// (construction.cpp:154-226) with the 64-bit string hashes (hash_algo 1 = aes64, the
// reference's pick on an x86 host with AES-NI; 3 = portable64).
inline std::vector<uint8_t> build(std::span<const std::string> keys, const ph_build_params& params,
                                  int hash_algo = 1, unsigned threads = 0, int device = 0,
                                  ph_build_stats* stats = nullptr) {
    std::vector<uint64_t> offsets(keys.size() + 1, 0);
    for (size_t i = 0; i < keys.size(); i++) offsets[i + 1] = offsets[i] + keys[i].size();
    std::vector<uint8_t> bytes(offsets.back() ? offsets.back() : 1);
    for (size_t i = 0; i < keys.size(); i++) std::copy(keys[i].begin(), keys[i].end(), bytes.begin() + offsets[i]);
    uint8_t* out_bytes = nullptr;
    size_t len = 0;
    check(ph_gpu_build_bytes(bytes.data(), offsets.data(), keys.size(), &params, hash_algo, threads, device,
                             &out_bytes, &len, stats));
    std::vector<uint8_t> out(out_bytes, out_bytes + len);
    ph_free(out_bytes);
    return out;
}

}  // namespace ph_gpu
