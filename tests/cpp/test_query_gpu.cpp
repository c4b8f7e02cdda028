// C++ parity test of the GPU query path through the C++ wrapper
// (include/ph_gpu/index.hpp), written after the reference's own query tests
// (/root/reference/proj/tests/test_query.cpp:23-117).
//
// The reference library (oracle/_ref/libptrhash_ref.so, test infrastructure)
// is dlopen'ed to build indexes and to produce the expected outputs; every
// GPU output must equal the reference's index_loop output exactly.
//
// Usage: test_query_gpu <path to libptrhash_ref.so>. Exit code 0 = all passed.
#include <dlfcn.h>
#include <unistd.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "ph_gpu/index.hpp"

namespace {

struct RefParams {
    uint32_t alpha_num, alpha_den, lambda_num, lambda_den;
    int32_t bucket_fn, remap_kind, reduce_kind;
    uint32_t max_seed_retries;
    uint64_t seed;
};

struct Ref {
    int (*preset)(const char*, RefParams*);
    int (*build_u64)(const uint64_t*, size_t, const RefParams*, unsigned, uint8_t**, size_t*);
    int (*build_bytes)(const uint8_t*, const uint64_t*, size_t, const RefParams*, unsigned,
                       uint8_t**, size_t*);
    void* (*load)(const uint8_t*, size_t);
    void (*unload)(void*);
    int (*query_u64)(const void*, const uint64_t*, size_t, uint64_t*, int, int, size_t, unsigned);
    int (*query_bytes)(const void*, const uint8_t*, const uint64_t*, size_t, uint64_t*, int, int,
                       size_t, unsigned);
    uint64_t (*index_u64)(const void*, uint64_t, int);
    uint64_t (*corpus_u64)(uint64_t, uint64_t);
    void (*free_)(void*);
};

int g_checks = 0, g_failed = 0;
#define CHECK(cond)                                                                 \
    do {                                                                            \
        g_checks++;                                                                 \
        if (!(cond)) {                                                              \
            g_failed++;                                                             \
            std::fprintf(stderr, "%s:%d: CHECK(%s) failed\n", __FILE__, __LINE__, #cond); \
        }                                                                           \
    } while (0)

template <class T>
void sym(void* lib, const char* name, T& f) {
    f = reinterpret_cast<T>(dlsym(lib, name));
    if (!f) {
        std::fprintf(stderr, "missing symbol %s\n", name);
        std::exit(2);
    }
}

std::vector<uint8_t> build(const Ref& R, const std::vector<uint64_t>& keys, const char* preset) {
    RefParams p;
    R.preset(preset, &p);
    uint8_t* b = nullptr;
    size_t n = 0;
    if (R.build_u64(keys.data(), keys.size(), &p, 0, &b, &n) != 0) std::exit(3);
    std::vector<uint8_t> v(b, b + n);
    R.free_(b);
    return v;
}

std::vector<uint64_t> corpus(const Ref& R, uint64_t n, uint64_t seed) {
    std::vector<uint64_t> k(n);
    for (uint64_t i = 0; i < n; i++) k[i] = R.corpus_u64(i, seed);
    return k;
}

bool is_bijection(std::vector<uint64_t> v, uint64_t n) {  // tests/oracles.hpp:73-79
    if (v.size() != n) return false;
    std::sort(v.begin(), v.end());
    for (uint64_t i = 0; i < n; i++)
        if (v[i] != i) return false;
    return true;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: %s <libptrhash_ref.so>\n", argv[0]);
        return 2;
    }
    void* lib = dlopen(argv[1], RTLD_NOW);
    if (!lib) {
        std::fprintf(stderr, "dlopen: %s\n", dlerror());
        return 2;
    }
    Ref R;
    sym(lib, "ref_preset", R.preset);
    sym(lib, "ref_build_u64", R.build_u64);
    sym(lib, "ref_build_bytes", R.build_bytes);
    sym(lib, "ref_load", R.load);
    sym(lib, "ref_unload", R.unload);
    sym(lib, "ref_query_u64", R.query_u64);
    sym(lib, "ref_query_bytes", R.query_bytes);
    sym(lib, "ref_index_u64", R.index_u64);
    sym(lib, "ref_corpus_u64", R.corpus_u64);
    sym(lib, "ref_free", R.free_);

    // construction through the C++ wrapper: ph_gpu::build gives the reference's bytes for the
    // same keys and preset (pilot search on the GPU and on host threads), and reports
    // duplicate keys like the reference's BuildError::kDuplicateKeys
    {
        const auto keys = corpus(R, 150'000, 5);
        for (const char* name : {"fast", "default", "compact"}) {
            const auto want = build(R, keys, name);
            for (const int mode : {2, 1}) {
                CHECK(ph_gpu_set_build_search(mode) == PH_OK);
                ph_build_stats st{};
                const auto got = ph_gpu::build(keys, ph_gpu::preset(name), 0, 0, &st);
                CHECK(got == want);
                CHECK(st.n == keys.size() && (st.reserved[0] == 1) == (mode == 2));
            }
        }
        CHECK(ph_gpu_set_build_search(0) == PH_OK);
        auto dup = keys;
        dup.back() = dup[3];
        bool threw = false;
        try {
            ph_gpu::build(dup, ph_gpu::preset("default"));
        } catch (const ph_gpu::Error& e) {
            threw = e.code() == PH_E_DUPLICATE;
        }
        CHECK(threw);
    }

    // test_query.cpp:23-49 — loop, batched and streaming agree elementwise, and
    // equal the reference, on a mix of member and non-member keys.
    {
        const uint64_t n = 200'000;
        const auto keys = corpus(R, n, 2);
        for (const char* name : {"fast", "default"}) {
            const auto bytes = build(R, keys, name);
            void* ref = R.load(bytes.data(), bytes.size());
            const ph_gpu::PtrHashIndex idx(bytes);
            auto queries = corpus(R, n, 777);
            for (uint64_t i = 0; i < n; i += 2) queries[i] = keys[i];
            for (const bool minimal : {true, false}) {
                std::vector<uint64_t> want(n);
                R.query_u64(ref, queries.data(), n, want.data(), minimal, 0, 0, 1);
                std::vector<uint64_t> loop(n);
                idx.index_loop(queries, loop.data(), minimal);
                CHECK(loop == want);
                for (const size_t batch : {size_t{1}, size_t{16}, size_t{64}, size_t{1000}}) {
                    std::vector<uint64_t> out(n);
                    idx.index_batched(queries, batch, out.data(), minimal);
                    CHECK(out == want);
                }
                for (const size_t ahead : {size_t{1}, size_t{32}, size_t{128}, n + 5}) {
                    std::vector<uint64_t> out(n);
                    idx.index_stream(queries, ahead, out.data(), minimal);
                    CHECK(out == want);
                }
                std::vector<uint32_t> o32(n);
                idx.index_u32(queries, o32.data(), minimal);
                bool same = true;
                for (uint64_t i = 0; i < n; i++) same &= o32[i] == static_cast<uint32_t>(want[i]);
                CHECK(same);
                idx.trim();  // cached scratch released; the next call allocates again
                std::vector<uint64_t> again(n);
                idx.index_loop(queries, again.data(), minimal);
                CHECK(again == want);
            }
            R.unload(ref);
        }
    }

    // test_query.cpp:51-64 — string query modes agree (+ bijection).
    {
        const uint64_t n = 30'000;
        std::vector<std::string> keys(n);
        uint64_t st = 9;
        for (auto& s : keys) {  // corpus_string-style lowercase keys, len 10..50
            st += 0x9e3779b97f4a7c15ULL;
            uint64_t z = R.corpus_u64(st, 9);
            s.resize(10 + z % 41);
            for (auto& c : s) {
                z = R.corpus_u64(z, 3);
                c = static_cast<char>('a' + z % 26);
            }
        }
        std::sort(keys.begin(), keys.end());
        keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
        std::vector<uint8_t> bytes;
        std::vector<uint64_t> offs{0};
        for (auto& s : keys) {
            bytes.insert(bytes.end(), s.begin(), s.end());
            offs.push_back(bytes.size());
        }
        RefParams p;
        R.preset("default", &p);
        uint8_t* b = nullptr;
        size_t blen = 0;
        if (R.build_bytes(bytes.data(), offs.data(), keys.size(), &p, 0, &b, &blen) != 0) return 3;
        std::vector<uint8_t> ptrh(b, b + blen);
        R.free_(b);
        // the same index built on the GPU through the C++ wrapper (aes64, the reference's pick here)
        if (ptrh[9] == 1) CHECK(ph_gpu::build(std::span<const std::string>(keys), ph_gpu::preset("default")) == ptrh);
        void* ref = R.load(ptrh.data(), ptrh.size());
        const ph_gpu::PtrHashIndex idx(ptrh);
        const size_t m = keys.size();
        std::vector<uint64_t> want(m), loop(m), batched(m), streamed(m);
        R.query_bytes(ref, bytes.data(), offs.data(), m, want.data(), 1, 0, 0, 1);
        idx.index_loop(keys, loop.data());
        idx.index_batched(keys, 32, batched.data());
        idx.index_stream(keys, 32, streamed.data());
        CHECK(loop == want);
        CHECK(batched == loop);
        CHECK(streamed == loop);
        CHECK(is_bijection(loop, m));
        CHECK(idx.index(std::string_view(keys[17])) == want[17]);
        R.unload(ref);
    }

    // test_query.cpp:66-74 — every query lands below n, member or not.
    {
        const uint64_t n = 100'000;
        const auto bytes = build(R, corpus(R, n, 4), "compact");
        const ph_gpu::PtrHashIndex idx(bytes);
        const auto q = corpus(R, 200'000, 70);
        std::vector<uint64_t> out(q.size());
        idx.index_stream(q, 32, out.data());
        CHECK(*std::max_element(out.begin(), out.end()) < n);
    }

    // test_query.cpp:76-84 — batched output equals single-key queries.
    {
        const uint64_t n = 10'000;
        const auto keys = corpus(R, n, 5);
        const auto bytes = build(R, keys, "fast");
        const ph_gpu::PtrHashIndex idx(bytes);
        std::vector<uint64_t> out(n);
        idx.index_batched(keys, 64, out.data());
        bool same = true;
        for (uint64_t i = 0; i < n; i += 37) same &= out[i] == idx.index(keys[i]);
        CHECK(same);
        void* ref = R.load(bytes.data(), bytes.size());
        CHECK(idx.index_no_remap(keys[3]) == R.index_u64(ref, keys[3], 0));
        R.unload(ref);
    }

    // test_query.cpp:86-92 — bijectivity through the streaming path.
    {
        const uint64_t n = 1'000'000;
        const auto keys = corpus(R, n, 6);
        const ph_gpu::PtrHashIndex idx(build(R, keys, "default"));
        std::vector<uint64_t> out(n);
        idx.index_stream(keys, 32, out.data());
        CHECK(is_bijection(out, n));
    }

    // test_serde.cpp (save_index / load_index round trip): an index loaded from a file
    // answers like the one created from the same bytes.
    {
        const uint64_t n = 50'000;
        const auto keys = corpus(R, n, 9);
        const auto bytes = build(R, keys, "default");
        const std::string path = "/tmp/ph_gpu_cpp_test_" + std::to_string(getpid()) + ".ptrh";
        FILE* f = std::fopen(path.c_str(), "wb");
        CHECK(f && std::fwrite(bytes.data(), 1, bytes.size(), f) == bytes.size());
        std::fclose(f);
        const auto loaded = ph_gpu::PtrHashIndex::load(path.c_str());
        std::remove(path.c_str());
        const ph_gpu::PtrHashIndex created(bytes);
        std::vector<uint64_t> a(n), b(n);
        loaded.index_stream(keys, 32, a.data());
        created.index_stream(keys, 32, b.data());
        CHECK(a == b && is_bijection(a, n));
        bool threw = false;
        try {
            ph_gpu::PtrHashIndex::load("/nonexistent/index.ptrh");
        } catch (const ph_gpu::Error&) {
            threw = true;
        }
        CHECK(threw);
    }

    // test_query.cpp:94-117 — threaded slices concatenate to the single-call answer
    // (one immutable handle shared by several host threads).
    {
        const uint64_t n = 300'000;
        const auto keys = corpus(R, n, 8);
        const ph_gpu::PtrHashIndex idx(build(R, keys, "default"));
        std::vector<uint64_t> single(n);
        idx.index_stream(keys, 32, single.data());
        for (const unsigned threads : {2u, 3u, 7u}) {
            std::vector<uint64_t> out(n);
            std::vector<std::thread> workers;
            const uint64_t chunk = n / threads + 1;
            for (unsigned w = 0; w < threads; w++) {
                workers.emplace_back([&, w] {
                    const uint64_t begin = std::min<uint64_t>(n, w * chunk);
                    const uint64_t end = std::min<uint64_t>(n, begin + chunk);
                    idx.index_stream(std::span(keys).subspan(begin, end - begin), 32,
                                     out.data() + begin);
                });
            }
            for (auto& t : workers) t.join();
            CHECK(out == single);
        }
    }

    // fused k-mer front end through the wrapper: identical to querying the materialised
    // k-mers (first base in the MSBs) with the reference
    {
        const uint64_t n_bases = 300'031;
        const int k = 31;
        std::vector<uint64_t> seq((n_bases + 31) / 32);
        for (uint64_t w = 0; w < seq.size(); w++) seq[w] = R.corpus_u64(w, 44);
        const uint64_t nw = n_bases - k + 1;
        std::vector<uint64_t> kmers(nw);
        for (uint64_t i = 0; i < nw; i++) {
            uint64_t v = 0;
            for (int t = 0; t < k; t++) {
                const uint64_t j = i + t;
                v = (v << 2) | ((seq[j / 32] >> (2 * (31 - j % 32))) & 3);
            }
            kmers[i] = v;
        }
        std::vector<uint64_t> uniq = kmers;
        std::sort(uniq.begin(), uniq.end());
        uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
        const auto bytes = build(R, uniq, "default");
        void* ref = R.load(bytes.data(), bytes.size());
        const ph_gpu::PtrHashIndex idx(bytes);
        std::vector<uint64_t> want(nw);
        R.query_u64(ref, kmers.data(), nw, want.data(), 1, 0, 0, 1);
        std::vector<uint32_t> got(nw);
        idx.index_kmers(seq.data(), n_bases, k, got.data());
        bool same = true;
        for (uint64_t i = 0; i < nw; i++) same &= got[i] == static_cast<uint32_t>(want[i]);
        CHECK(same);
        R.unload(ref);
    }

    // key-kind mismatch is an error at the C ABI (the reference would misuse silently)
    {
        const auto keys = corpus(R, 1000, 11);
        const ph_gpu::PtrHashIndex idx(build(R, keys, "fast"));
        bool threw = false;
        try {
            std::vector<std::string> s{"abc"};
            std::vector<uint64_t> o(1);
            idx.index_loop(s, o.data());
        } catch (const ph_gpu::Error& e) {
            threw = e.code() == PH_E_KEYKIND;
        }
        CHECK(threw);
    }

    std::printf("test_query_gpu: %d checks, %d failed, %llu kernel launches\n", g_checks, g_failed,
                static_cast<unsigned long long>(ph_gpu_launch_count()));
    return g_failed ? 1 : 0;
}
