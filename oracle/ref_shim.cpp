// TEST INFRASTRUCTURE ONLY — a C ABI over the UNMODIFIED reference library
// (/root/reference/proj), so pytest (ctypes) and bench.py's reference arm can
// drive the reference builder and its CPU query path. Never linked into the
// product (paper_2502_15539_b200/libph_gpu.so).
//
// Every entry point forwards to a reference symbol:
//   build / build_with_shape     proj/src/construction.cpp:139-152
//   build_sharded (KeySource)    proj/src/sharding.cpp:305-327, KeySource sharding.hpp:44-51
//   serialize / deserialize      proj/src/serde.cpp:142-240
//   index / index_no_remap       proj/include/ptrhash/index.hpp:60-64
//   index_loop/batched/stream    proj/src/index.cpp:15-137
//   threaded slices              proj/tools/ptrhash.cpp:486-512 (chunk = n/T + 1)
//   hash/gamma/reduce/clef prims hash.hpp:27-32, hash.cpp:159, bucket_fn.hpp:49-72,
//                                reduce.hpp:27-77, cacheline_ef.cpp:33-65
//   build-attempt front phases   construction.cpp:28-60,98-111; engine.hpp:412-518

#include <atomic>
#include <cstdlib>
#include <cstring>
#include <string>
#include <string_view>
#include <thread>
#include <vector>

#include "ptrhash/build.hpp"
#include "ptrhash/bucket_fn.hpp"
#include "ptrhash/cacheline_ef.hpp"
#include "ptrhash/corpus.hpp"
#include "ptrhash/elias_fano.hpp"
#include "ptrhash/index.hpp"
#include "ptrhash/serde.hpp"
#include "ptrhash/sharding.hpp"
#include "ptrhash/kernels.hpp"
#include "engine.hpp"  // proj/src: detail::H64, detail::scatter_to_parts

using namespace ptrhash;

namespace {

thread_local std::string g_err;

struct RefParams {
    uint32_t alpha_num, alpha_den, lambda_num, lambda_den;
    int32_t bucket_fn, remap_kind, reduce_kind;
    uint32_t max_seed_retries;
    uint64_t seed;
};

BuildParams to_params(const RefParams* p) {
    BuildParams bp;
    bp.alpha = {p->alpha_num, p->alpha_den};
    bp.lambda = {p->lambda_num, p->lambda_den};
    bp.bucket_fn = static_cast<BucketFnKind>(p->bucket_fn);
    bp.remap_kind = static_cast<RemapKind>(p->remap_kind);
    bp.reduce_kind = static_cast<ReduceKind>(p->reduce_kind);
    bp.max_seed_retries = p->max_seed_retries;
    bp.seed = p->seed;
    return bp;
}

int emit(const PtrHashIndex& idx, uint8_t** out, size_t* out_len) {
    std::vector<uint8_t> bytes = serialize(idx);
    *out = static_cast<uint8_t*>(std::malloc(bytes.size() ? bytes.size() : 1));
    if (!*out) {
        g_err = "out of memory";
        return -1;
    }
    std::memcpy(*out, bytes.data(), bytes.size());
    *out_len = bytes.size();
    return 0;
}

template <class F>
int guarded(F&& f) {
    try {
        return f();
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// Concatenated byte buffer + offsets[n+1] as a reference KeySource.
class ConcatSource final : public KeySource {
  public:
    ConcatSource(const uint8_t* data, const uint64_t* offsets, uint64_t n)
        : data_(data), offsets_(offsets), n_(n) {}
    uint64_t size() const override { return n_; }
    KeyKind kind() const override { return KeyKind::kBytes; }
    void for_each_str(const std::function<void(std::string_view)>& fn) const override {
        for (uint64_t i = 0; i < n_; i++)
            fn(std::string_view(reinterpret_cast<const char*>(data_) + offsets_[i],
                                offsets_[i + 1] - offsets_[i]));
    }

  private:
    const uint8_t* data_;
    const uint64_t* offsets_;
    uint64_t n_;
};

std::vector<std::string> to_strings(const uint8_t* data, const uint64_t* offsets, size_t b,
                                    size_t e) {
    std::vector<std::string> v;
    v.reserve(e - b);
    for (size_t i = b; i < e; i++)
        v.emplace_back(reinterpret_cast<const char*>(data) + offsets[i], offsets[i + 1] - offsets[i]);
    return v;
}

template <class Body>
void run_slices(size_t n, unsigned threads, Body&& body) {
    if (threads <= 1) {
        body(size_t{0}, n);
        return;
    }
    std::vector<std::thread> workers;
    const size_t chunk = n / threads + 1;  // proj/tools/ptrhash.cpp:488
    for (unsigned w = 0; w < threads; w++) {
        workers.emplace_back([&, w] {
            const size_t begin = std::min<size_t>(n, size_t{w} * chunk);
            const size_t end = std::min<size_t>(n, begin + chunk);
            if (begin < end) body(begin, end);
        });
    }
    for (auto& t : workers) t.join();
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
void ref_free(void* p) { std::free(p); }
int ref_cpu_has_aes() { return cpu_has_aes() ? 1 : 0; }
unsigned ref_hw_threads() { return std::thread::hardware_concurrency(); }

int ref_preset(const char* name, RefParams* out) {
    return guarded([&] {
        BuildParams p = preset(name);
        out->alpha_num = p.alpha.num;
        out->alpha_den = p.alpha.den;
        out->lambda_num = p.lambda.num;
        out->lambda_den = p.lambda.den;
        out->bucket_fn = static_cast<int32_t>(p.bucket_fn);
        out->remap_kind = static_cast<int32_t>(p.remap_kind);
        out->reduce_kind = static_cast<int32_t>(p.reduce_kind);
        out->max_seed_retries = p.max_seed_retries;
        out->seed = p.seed;
        return 0;
    });
}

int ref_compute_shape(uint64_t n, const RefParams* p, uint64_t* P, uint64_t* S, uint64_t* B) {
    return guarded([&] {
        Shape s = compute_shape(n, to_params(p));
        *P = s.parts;
        *S = s.slots_per_part;
        *B = s.buckets_per_part;
        return 0;
    });
}

int ref_build_u64(const uint64_t* keys, size_t n, const RefParams* p, unsigned threads,
                  uint8_t** out, size_t* out_len) {
    return guarded([&] {
        PtrHashIndex idx = build(std::span<const uint64_t>(keys, n), to_params(p), threads);
        return emit(idx, out, out_len);
    });
}

int ref_build_u64_shape(const uint64_t* keys, size_t n, const RefParams* p, uint64_t P,
                        uint64_t S, uint64_t B, unsigned threads, uint8_t** out,
                        size_t* out_len) {
    return guarded([&] {
        Shape s;
        s.n = n;
        s.parts = P;
        s.slots_per_part = S;
        s.buckets_per_part = B;
        PtrHashIndex idx =
            build_with_shape(std::span<const uint64_t>(keys, n), to_params(p), s, threads);
        return emit(idx, out, out_len);
    });
}

// build() with BuildStats: also returns bucket_size_counts (stats.cpp:59-61).
int ref_build_u64_stats(const uint64_t* keys, size_t n, const RefParams* p, unsigned threads,
                        uint8_t** out, size_t* out_len, uint64_t* sizes, size_t cap,
                        size_t* sizes_len) {
    return guarded([&] {
        BuildStats st;
        PtrHashIndex idx = build(std::span<const uint64_t>(keys, n), to_params(p), threads, &st);
        *sizes_len = st.bucket_size_counts.size();
        for (size_t i = 0; i < cap && i < st.bucket_size_counts.size(); i++)
            sizes[i] = st.bucket_size_counts[i];
        return emit(idx, out, out_len);
    });
}

// build(span<std::string>) — the reference's string builder (memory heavy).
int ref_build_bytes(const uint8_t* data, const uint64_t* offsets, size_t n, const RefParams* p,
                    unsigned threads, uint8_t** out, size_t* out_len) {
    return guarded([&] {
        std::vector<std::string> keys = to_strings(data, offsets, 0, n);
        PtrHashIndex idx = build(std::span<const std::string>(keys), to_params(p), threads);
        return emit(idx, out, out_len);
    });
}

// build_sharded over the concatenated buffer (memory lean; one shard when
// n < 2^32 gives the same index as build(), SURVEY §7 hard parts).
int ref_build_bytes_lean(const uint8_t* data, const uint64_t* offsets, size_t n,
                         const RefParams* p, unsigned threads, uint8_t** out, size_t* out_len) {
    return guarded([&] {
        ConcatSource src(data, offsets, n);
        ShardPlan plan;
        PtrHashIndex idx = build_sharded(src, to_params(p), plan, threads);
        return emit(idx, out, out_len);
    });
}

void* ref_load(const uint8_t* bytes, size_t len) {
    try {
        return new PtrHashIndex(deserialize(std::span<const uint8_t>(bytes, len)));
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

void ref_unload(void* h) { delete static_cast<PtrHashIndex*>(h); }

uint64_t ref_index_u64(const void* h, uint64_t key, int minimal) {
    const auto* idx = static_cast<const PtrHashIndex*>(h);
    return minimal ? idx->index(key) : idx->index_no_remap(key);
}

uint64_t ref_index_bytes1(const void* h, const uint8_t* p, size_t len, int minimal) {
    const auto* idx = static_cast<const PtrHashIndex*>(h);
    std::string_view s(reinterpret_cast<const char*>(p), len);
    return minimal ? idx->index(s) : idx->index_no_remap(s);
}

// mode: 0 = index_loop, 1 = index_batched(width), 2 = index_stream(width)
int ref_query_u64(const void* h, const uint64_t* keys, size_t n, uint64_t* out, int minimal,
                  int mode, size_t width, unsigned threads) {
    return guarded([&] {
        const auto* idx = static_cast<const PtrHashIndex*>(h);
        run_slices(n, threads, [&](size_t b, size_t e) {
            std::span<const uint64_t> ks(keys + b, e - b);
            if (mode == 0) idx->index_loop(ks, out + b, minimal != 0);
            else if (mode == 1) idx->index_batched(ks, width, out + b, minimal != 0);
            else idx->index_stream(ks, width, out + b, minimal != 0);
        });
        return 0;
    });
}

// mode 3 = single-key index(string_view) loop over the concatenated buffer
// (no std::string materialisation); 0/1/2 materialise std::strings per slice
// and call index_loop / index_batched / index_stream.
int ref_query_bytes(const void* h, const uint8_t* data, const uint64_t* offsets, size_t n,
                    uint64_t* out, int minimal, int mode, size_t width, unsigned threads) {
    return guarded([&] {
        const auto* idx = static_cast<const PtrHashIndex*>(h);
        run_slices(n, threads, [&](size_t b, size_t e) {
            if (mode == 3) {
                for (size_t i = b; i < e; i++) {
                    std::string_view s(reinterpret_cast<const char*>(data) + offsets[i],
                                       offsets[i + 1] - offsets[i]);
                    out[i] = minimal ? idx->index(s) : idx->index_no_remap(s);
                }
                return;
            }
            std::vector<std::string> ks = to_strings(data, offsets, b, e);
            std::span<const std::string> sp(ks);
            if (mode == 0) idx->index_loop(sp, out + b, minimal != 0);
            else if (mode == 1) idx->index_batched(sp, width, out + b, minimal != 0);
            else idx->index_stream(sp, width, out + b, minimal != 0);
        });
        return 0;
    });
}

// Pre-materialised std::string keys (so a timed index_loop / index_batched / index_stream
// over span<const std::string> excludes building the strings; bench.py's CPU matrix).
void* ref_strings_new(const uint8_t* data, const uint64_t* offsets, size_t n) {
    try {
        return new std::vector<std::string>(to_strings(data, offsets, 0, n));
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}
void ref_strings_free(void* s) { delete static_cast<std::vector<std::string>*>(s); }
// mode: 0 = index_loop, 1 = index_batched(width), 2 = index_stream(width), over T slices
int ref_query_strings(const void* h, const void* strs, uint64_t* out, int minimal, int mode,
                      size_t width, unsigned threads) {
    return guarded([&] {
        const auto* idx = static_cast<const PtrHashIndex*>(h);
        const auto& v = *static_cast<const std::vector<std::string>*>(strs);
        run_slices(v.size(), threads, [&](size_t b, size_t e) {
            std::span<const std::string> sp(v.data() + b, e - b);
            if (mode == 0) idx->index_loop(sp, out + b, minimal != 0);
            else if (mode == 1) idx->index_batched(sp, width, out + b, minimal != 0);
            else idx->index_stream(sp, width, out + b, minimal != 0);
        });
        return 0;
    });
}

// ---- primitives for known-answer tests ----
uint64_t ref_mix_constant_inverse() { return mix_constant_inverse(); }
uint64_t ref_hash_int(uint64_t k, uint64_t seed) { return hash_int(k, seed); }
uint64_t ref_hash_pilot(uint64_t p, uint64_t seed) { return hash_pilot(p, seed); }
void ref_hash_bytes(const uint8_t* p, size_t len, uint64_t seed, int algo, uint64_t* hi,
                    uint64_t* lo) {
    HashValue v = hash_bytes(p, len, seed, static_cast<HashAlgo>(algo));
    *hi = v.hi;
    *lo = v.lo;
}
uint64_t ref_gamma(int kind, uint64_t x) { return gamma_eval(static_cast<BucketFnKind>(kind), x); }
uint64_t ref_reduce(uint64_t S, uint64_t x) { return Reducer(S).reduce(x); }
void ref_fastmod_magic(uint64_t S, uint64_t* hi, uint64_t* lo) {
    FastModU64 m = FastModU64::make(S);
    *hi = m.magic_hi;
    *lo = m.magic_lo;
}
void ref_part_and_bucket(uint64_t h, uint64_t P, uint64_t B, int fn, uint64_t* part,
                         uint64_t* bucket) {
    Shape s;
    s.parts = P;
    s.buckets_per_part = B;
    PartAndBucket pb = part_and_bucket(h, s, static_cast<BucketFnKind>(fn));
    *part = pb.part;
    *bucket = pb.bucket;
}
int ref_clef_encode(const uint64_t* v, size_t n, uint8_t* out64) {
    CacheLineEfBlock b;
    ClefStatus st = clef_encode(std::span<const uint64_t>(v, n), b);
    std::memcpy(out64, b.bytes.data(), 64);
    return static_cast<int>(st);
}
uint64_t ref_clef_get(const uint8_t* block64, size_t i) {
    CacheLineEfBlock b;
    std::memcpy(b.bytes.data(), block64, 64);
    return clef_get(b, i);
}
uint64_t ref_corpus_u64(uint64_t i, uint64_t gen_seed) { return corpus_u64(i, gen_seed); }

// The data-parallel front of one u64 build attempt, with the reference's own code:
// hash_all (construction.cpp:98-111: kernels::active_ops().hash_u64 into detail::H64),
// detail::scatter_to_parts (engine.hpp:412-474) and each part's std::sort + duplicate check
// (engine.hpp:505-518). Returns 0 ok, 1 kOversubscribed, 2 kDuplicateHashes, -1 error;
// hashes_out[n] part-major and sorted, offsets_out[P+1].
int ref_build_prepare_u64(const uint64_t* keys, size_t n, uint64_t P, uint64_t S, uint64_t seed,
                          unsigned threads, uint64_t* hashes_out, uint64_t* offsets_out) {
    return guarded([&] {
        Shape shape;
        shape.n = n;
        shape.parts = P;
        shape.slots_per_part = S;
        std::vector<detail::H64> h(n);
        kernels::active_ops().hash_u64(keys, n, seed, reinterpret_cast<uint64_t*>(h.data()));
        std::vector<uint64_t> offsets;
        const auto f = detail::scatter_to_parts<detail::H64>(
            shape, h, 0, P, detail::effective_threads(threads), offsets);
        if (f == detail::AttemptFail::kOversubscribed) return 1;
        // parts sorted in parallel, as build_parts does (engine.hpp:484-518)
        std::atomic<uint64_t> next{0};
        std::atomic<int> status{0};
        std::vector<std::thread> workers;
        const unsigned t = detail::effective_threads(threads);
        for (unsigned w = 0; w < t; w++)
            workers.emplace_back([&] {
                for (uint64_t p; (p = next.fetch_add(1)) < P;) {
                    auto b = h.begin() + offsets[p], e = h.begin() + offsets[p + 1];
                    std::sort(b, e);
                    for (auto it = b; it != e && it + 1 != e; ++it)
                        if (*it == *(it + 1)) status = 2;
                }
            });
        for (auto& th : workers) th.join();
        std::memcpy(hashes_out, h.data(), n * 8);
        std::memcpy(offsets_out, offsets.data(), (P + 1) * 8);
        return status.load();
    });
}

}  // extern "C"
