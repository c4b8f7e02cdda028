// ph_abi.cu — host side of the C ABI (include/ph_gpu.h).
//
//  * PTRH v1 parsing and validation, mirroring deserialize()
//    (/root/reference/proj/src/serde.cpp:176-240) check for check;
//  * device upload: pilots and CacheLineEF/plain32 payload byte-identical to
//    the file; Elias-Fano's three u64 arrays re-aligned (serde.cpp:93-101);
//    the optimal-gamma table computed on the host exactly as
//    bucket_fn.cpp:16-39 does (double ln, monotone clamp) and uploaded;
//  * the query entry points: device-resident (async) and host-resident
//    (pipelined H2D -> kernel -> D2H over chunks and streams, synchronous).
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/ph_gpu.h"
#include "ph_device.cuh"
#include "ph_kernels.h"
#include "ph_nvtx.h"

using u128 = unsigned __int128;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}
int cuda_fail(cudaError_t e, const char* what) {
    return fail(PH_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define PH_CUDA(call)                                 \
    do {                                              \
        cudaError_t e_ = (call);                      \
        if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
    } while (0)

uint64_t le64(const uint8_t* p) {
    uint64_t v;
    std::memcpy(&v, p, 8);
    return v;
}
uint32_t le32(const uint8_t* p) {
    uint32_t v;
    std::memcpy(&v, p, 4);
    return v;
}
bool is_pow2(uint64_t x) { return x && !(x & (x - 1)); }

// Sets the device for the scope of one ABI call and restores the caller's.
struct DeviceGuard {
    int prev = -1;
    cudaError_t err = cudaSuccess;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) err = cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

// bucket_fn.cpp:16-39 — filled with double-precision ln, monotonized.
void optimal_table(std::vector<uint64_t>& t) {
    t.resize(65537);
    const double eps = 1.0 / 256.0;
    const double scale = std::ldexp(1.0, 64);
    uint64_t prev = 0;
    for (size_t i = 0; i <= 65536; i++) {
        const double x = static_cast<double>(i) / 65536;
        double y = x;
        if (x < 1.0) y = x + (1.0 - eps) * (1.0 - x) * std::log(1.0 - x);
        const double scaled = y * scale;
        uint64_t u;
        if (scaled >= scale) u = UINT64_MAX;
        else if (scaled <= 0.0) u = 0;
        else u = static_cast<uint64_t>(scaled);
        if (u < prev) u = prev;
        t[i] = u;
        prev = u;
    }
}

// Hot-first pilot layout budget: the first hot_bytes/P pilots of every
// part go to a contiguous hot region under a persisting L2 window.
constexpr uint64_t kDefaultHotBytes = uint64_t{64} << 20;
// ph_gpu_index_set_l2_policy flags
constexpr int kL2ColdEvictFirst = 1;  // cold-region pilot loads use L2::evict_first
constexpr int kL2NoWindow = 2;        // no persisting access-policy window
constexpr int kDefaultL2Flags = 0;

}  // namespace

namespace phg {
// for ph_builder.cu: the thread-local error of this ABI, and the optimal-gamma table
int report_error(int code, const std::string& msg) { return fail(code, msg); }
void optimal_gamma_table(std::vector<uint64_t>& t) { optimal_table(t); }
}  // namespace phg

namespace {
struct Pipeline;
}

struct ph_gpu_index {
    int device = 0;
    int sms = 148;
    ph_gpu_info info{};
    phg::DevIndex dev{};
    void* d_pilots = nullptr;
    void* d_remap = nullptr;
    void* d_ef[3] = {nullptr, nullptr, nullptr};
    void* d_opt = nullptr;
    void* d_aes = nullptr;  // AES T-tables (string indexes, small batches)
    cudaMemPool_t pool = nullptr;  // stream-ordered scratch for the deferred remap
    // host-path pipelines (streams + staging buffers), reused across calls
    mutable std::mutex pl_mu;
    mutable std::vector<Pipeline*> pl_cache;
    void (*pl_free)(ph_gpu_index*) = nullptr;  // frees pl_cache (set at create)
    // single-key queries (index() / index_no_remap()): one block of mapped pinned host
    // memory (key, offsets, output, key bytes) the kernel reads and writes in place, and
    // one stream, reused under single_mu: no allocation or copy call per query
    mutable std::mutex single_mu;
    mutable uint8_t* single_h = nullptr;
    mutable uint8_t* single_d = nullptr;  // device alias of single_h
    mutable size_t single_cap = 0;
    mutable cudaStream_t single_s = nullptr;
};

namespace {

// PTRH v1 (serde.hpp:12-31) -> validated header + payload views.
struct Parsed {
    uint8_t key_kind, algo, bucket_fn, remap_kind, reduce_kind;
    uint64_t n, P, S, B, seed, pilots_len, remap_len;
    const uint8_t* pilots;
    const uint8_t* remap;
    // Elias-Fano
    uint64_t ef_count = 0, ef_universe = 0;
    uint8_t ef_low_bits = 0;
    std::vector<uint64_t> ef[3];
};

int parse_ptrh(const uint8_t* b, size_t len, Parsed& p) {
    if (!b) return fail(PH_E_INVALID, "null index bytes");
    if (len < 4) return fail(PH_E_FORMAT, "index file truncated");
    if (std::memcmp(b, "PTRH", 4) != 0) return fail(PH_E_FORMAT, "not an index file (bad magic)");
    if (len < 72) return fail(PH_E_FORMAT, "index file truncated");
    const uint32_t version = le32(b + 4);
    if (version != 1)
        return fail(PH_E_FORMAT, "unsupported index format version " + std::to_string(version));
    p.key_kind = b[8];
    p.algo = b[9];
    p.bucket_fn = b[10];
    p.remap_kind = b[11];
    p.reduce_kind = b[12];
    if (p.key_kind > 1) return fail(PH_E_FORMAT, "unknown key kind id");
    if (p.algo > 4) return fail(PH_E_FORMAT, "unknown hash algorithm id");
    if (p.bucket_fn > 4) return fail(PH_E_FORMAT, "unknown bucket function id");
    if (p.remap_kind > 2) return fail(PH_E_FORMAT, "unknown remap kind id");
    if (p.reduce_kind > 2) return fail(PH_E_FORMAT, "unknown reduce kind id");
    // No AES-NI requirement (serde.cpp:200-202): the GPU computes AES itself.
    p.n = le64(b + 16);
    p.P = le64(b + 24);
    p.S = le64(b + 32);
    p.B = le64(b + 40);
    p.seed = le64(b + 48);
    p.pilots_len = le64(b + 56);
    p.remap_len = le64(b + 64);
    if (p.n == 0 || p.P == 0 || p.S == 0) return fail(PH_E_FORMAT, "index file: degenerate shape");
    if ((u128)p.P * p.S > ((u128)1 << 62) || (u128)p.P * p.B > ((u128)1 << 62))
        return fail(PH_E_FORMAT, "index file: shape out of range");
    if (p.n > p.P * p.S) return fail(PH_E_FORMAT, "index file: n exceeds the slot count");
    if (p.pilots_len != p.P * p.B)
        return fail(PH_E_FORMAT, "index file: pilot length does not match shape");
    if ((u128)(len - 72) != (u128)p.pilots_len + p.remap_len)
        return fail(PH_E_FORMAT, "index file: payload length mismatch");
    p.pilots = b + 72;
    p.remap = b + 72 + p.pilots_len;
    const uint64_t count = p.P * p.S - p.n;
    switch (p.remap_kind) {
        case 0:
            if (p.remap_len != count * 4) return fail(PH_E_FORMAT, "index file: bad plain remap length");
            break;
        case 1:
            if (p.remap_len != (count + 43) / 44 * 64)
                return fail(PH_E_FORMAT, "index file: bad cacheline-ef remap length");
            break;
        case 2: {  // serde.cpp:119-136
            size_t pos = 0;
            auto need = [&](size_t k) { return pos + k <= p.remap_len; };
            if (!need(17)) return fail(PH_E_FORMAT, "index file truncated");
            p.ef_count = le64(p.remap);
            p.ef_universe = le64(p.remap + 8);
            p.ef_low_bits = p.remap[16];
            pos = 17;
            if (p.ef_count != count) return fail(PH_E_FORMAT, "index file: bad elias-fano count");
            for (int a = 0; a < 3; a++) {
                if (!need(8)) return fail(PH_E_FORMAT, "index file truncated");
                const uint64_t m = le64(p.remap + pos);
                pos += 8;
                if (m > p.remap_len / 8 + 1)
                    return fail(PH_E_FORMAT, "index file: array length out of range");
                if (!need(m * 8)) return fail(PH_E_FORMAT, "index file truncated");
                p.ef[a].resize(m);
                for (uint64_t i = 0; i < m; i++) p.ef[a][i] = le64(p.remap + pos + 8 * i);
                pos += m * 8;
            }
            if (pos != p.remap_len) return fail(PH_E_FORMAT, "index file: trailing bytes");
            if (count > 0 && (p.ef[2].empty() || p.ef[1].empty()))
                return fail(PH_E_FORMAT, "index file: bad elias-fano payload");
            break;
        }
    }
    if (!is_pow2(p.S) && p.S >= (uint64_t{1} << 32))
        return fail(PH_E_FORMAT, "reduce: fastmod needs S < 2^32");  // reduce.hpp:56-57
    return PH_OK;
}

int upload(const void* src, size_t bytes, void** dst) {
    *dst = nullptr;
    if (bytes == 0) return PH_OK;
    cudaError_t e = cudaMalloc(dst, bytes);
    if (e != cudaSuccess) return fail(PH_E_NOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    e = cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy(upload)");
    return PH_OK;
}

// Single-key scratch (caller holds single_mu; the index's device is current).
constexpr size_t kSingleHeader = 64;  // [0] key / offsets[2] at 0..15, output at 16
int ensure_single(const ph_gpu_index* ix, size_t key_bytes) {
    const size_t need = kSingleHeader + ((key_bytes + 15) & ~size_t{15}) + 16;
    if (!ix->single_s) {
        cudaError_t e = cudaStreamCreateWithFlags(&ix->single_s, cudaStreamNonBlocking);
        if (e != cudaSuccess) return cuda_fail(e, "single-key stream");
    }
    if (ix->single_cap >= need) return PH_OK;
    if (ix->single_h) cudaFreeHost(ix->single_h);
    ix->single_h = ix->single_d = nullptr;
    ix->single_cap = 0;
    size_t cap = need < 4096 ? 4096 : need * 2;
    void* h = nullptr;
    cudaError_t e = cudaHostAlloc(&h, cap, cudaHostAllocMapped);
    if (e != cudaSuccess) return fail(PH_E_NOMEM, "single-key scratch (mapped pinned memory)");
    void* d = nullptr;
    e = cudaHostGetDevicePointer(&d, h, 0);
    if (e != cudaSuccess) {
        cudaFreeHost(h);
        return cuda_fail(e, "cudaHostGetDevicePointer");
    }
    std::memset(h, 0, cap);
    ix->single_h = static_cast<uint8_t*>(h);
    ix->single_d = static_cast<uint8_t*>(d);
    ix->single_cap = cap;
    return PH_OK;
}
void free_single(ph_gpu_index* ix) {
    if (ix->single_s) cudaStreamSynchronize(ix->single_s);
    if (ix->single_h) cudaFreeHost(ix->single_h);
    if (ix->single_s) cudaStreamDestroy(ix->single_s);
    ix->single_h = ix->single_d = nullptr;
    ix->single_s = nullptr;
}

// The device-wide persisting-L2 set-aside is shared by every index on a device: each live
// index registers the set-aside its window wants (0: none), and the device limit is the
// largest wanted by any of them, so creating or re-laying out one index never cancels
// another's window. (Consequence, documented in ph_gpu.h: while an index with a window is
// live, the partitioned path of a DRAM-sized index runs with that set-aside in place.)
std::mutex g_l2_mu;
std::map<int, std::map<const ph_gpu_index*, size_t>> g_l2_wants;

// Sets this device's limit to the largest registered want; returns the limit now in force.
size_t l2_apply_limit_locked(int device) {
    size_t want = 0;
    for (const auto& kv : g_l2_wants[device]) want = kv.second > want ? kv.second : want;
    size_t cur = 0;
    cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
    if (cur != want && cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want) != cudaSuccess)
        cudaGetLastError();
    cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
    return cur;
}

void l2_unregister(const ph_gpu_index* ix) {
    std::lock_guard<std::mutex> lk(g_l2_mu);
    auto& m = g_l2_wants[ix->device];
    if (m.erase(ix)) l2_apply_limit_locked(ix->device);
}

// Uploads the file-order pilots `file` (P*B bytes) in the hot-first layout for `hot_bytes`
// and sets the persisting-L2 window over the hot region. The new device buffer is built
// first; only when it is complete does it replace the index's pilots and layout fields, so
// a failure leaves the index as it was.
int apply_pilot_layout(ph_gpu_index* ix, const uint8_t* file, uint64_t hot_bytes, int flags) {
    const uint64_t P = ix->info.parts, B = ix->info.buckets_per_part;
    const uint64_t total = P * B;
    uint64_t H = B;  // hot_bytes == 0 or everything fits: the file's own order
    if (hot_bytes && total > hot_bytes && P > 0) H = hot_bytes / P < B ? hot_bytes / P : B;
    void* buf = nullptr;
    int rc = upload(file, total, &buf);  // file order
    if (rc) {
        cudaFree(buf);
        return rc;
    }
    if (H != B) {  // permute to the hot-first layout on the device (k_relayout)
        void* lay = nullptr;
        cudaError_t e = cudaMalloc(&lay, total);
        if (e != cudaSuccess) {
            cudaFree(buf);
            return fail(PH_E_NOMEM, "cudaMalloc(pilot layout)");
        }
        e = phg::launch_relayout(static_cast<const uint8_t*>(buf), static_cast<uint8_t*>(lay), P,
                                 B, H, nullptr);
        if (e == cudaSuccess) e = cudaStreamSynchronize(nullptr);
        cudaFree(buf);
        if (e != cudaSuccess) {
            cudaFree(lay);
            return cuda_fail(e, "pilot relayout");
        }
        buf = lay;
    }
    // the window this layout wants (0: none)
    uint64_t win = 0;
    size_t want = 0;
    if (!(flags & kL2NoWindow) && hot_bytes) {
        int max_window = 0, max_persist = 0;
        cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, ix->device);
        cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, ix->device);
        if (max_window > 0 && max_persist > 0 && P * H > 0) {
            win = P * H < (uint64_t)max_window ? P * H : (uint64_t)max_window;
            want = win < (uint64_t)max_persist ? win : (uint64_t)max_persist;
        }
    }
    // swap in the new layout
    phg::DevIndex& d = ix->dev;
    if (ix->d_pilots) {
        cudaDeviceSynchronize();  // (set_l2_policy: no query may still read the old buffer)
        cudaFree(ix->d_pilots);
    }
    ix->d_pilots = buf;
    d.pilots = static_cast<const uint8_t*>(buf);
    d.hot_b = H;
    d.cold_b = B - H;
    d.hot_total = P * H;
    d.cold_evict_first = (flags & kL2ColdEvictFirst) ? 1 : 0;
    d.window_bytes = 0;
    d.window_hit_ratio = 0.f;
    std::lock_guard<std::mutex> lk(g_l2_mu);
    auto& wants = g_l2_wants[ix->device];
    wants[ix] = want;
    // Lines left persisting by earlier windowed launches would keep their share of the L2
    // (the partitioned path's pass B needs all of it): reset them only when no live index
    // on this device has a window that relies on them.
    bool other_window = false;
    for (const auto& kv : wants) other_window |= kv.first != ix && kv.second > 0;
    if (!other_window) cudaCtxResetPersistingL2Cache();
    const size_t cur = l2_apply_limit_locked(ix->device);
    if (win && cur > 0) {
        d.window_bytes = win;
        d.window_hit_ratio = cur >= win ? 1.f : static_cast<float>(cur) / static_cast<float>(win);
    }
    return PH_OK;
}

void release(ph_gpu_index* ix) {
    if (!ix) return;
    DeviceGuard g(ix->device);
    l2_unregister(ix);
    free_single(ix);
    if (ix->pl_free) ix->pl_free(ix);
    cudaFree(ix->d_pilots);
    cudaFree(ix->d_remap);
    for (void* p : ix->d_ef) cudaFree(p);
    cudaFree(ix->d_opt);
    cudaFree(ix->d_aes);
    if (ix->pool) cudaMemPoolDestroy(ix->pool);
    delete ix;
}

// Stream-ordered scratch for the deferred remap list of one launch: used
// for minimal queries of at least kDeferMin keys; capacity n/32 + 64 Ki entries (3x the
// 1% remap rate of alpha = 0.99; overflow entries are decoded inline, never dropped).
std::atomic<uint64_t> g_defer_min{uint64_t{1} << 20};  // ph_gpu_set_defer_min

struct DeferScratch {
    phg::RemapList rl{nullptr, nullptr, nullptr, 0};
    void* p = nullptr;
    cudaStream_t s;
    DeferScratch(const ph_gpu_index* ix, uint64_t n, int minimal, cudaStream_t stream) : s(stream) {
        if (!minimal || n < g_defer_min.load() || !ix->pool) return;
        const uint64_t cap = n / 32 + 65536;
        const size_t counts_bytes = size_t{phg::kMaxRemapLists} * 4;
        if (cudaMallocFromPoolAsync(&p, counts_bytes + cap * 16, ix->pool, s) != cudaSuccess) {
            cudaGetLastError();
            p = nullptr;
            return;  // inline remap
        }
        auto* b = static_cast<uint8_t*>(p);
        rl.counts = reinterpret_cast<uint32_t*>(b);  // every grid warp writes its count
        rl.idx = reinterpret_cast<uint64_t*>(b + counts_bytes);
        rl.rem = rl.idx + cap;
        rl.cap = cap;
    }
    ~DeferScratch() {
        if (p) cudaFreeAsync(p, s);
    }
};

// Partitioned path (ph_partition.cu): for DRAM-sized pilot arrays and large
// device-resident batches, keys are binned into G hash groups whose pilot slices (32 MiB
// each) stay L2-resident while pass B answers them group after group, then un-permuted.
// It needs the file-order pilot layout without a persisting set-aside (the default for
// DRAM-sized arrays); "auto" uses it for batches of at least pilot_bytes / 32 keys (u64 keys
// and k-mer windows): the break-even against the direct kernel is ~1e7 keys at config 3
// (profiles/r01_partition_batch_sizes.txt). At 1e9 keys: 10.2 ms against 15.3 ms for the
// direct kernel on the hot-first layout; config 5 (k-mers) 10.8 ms against 13.9 ms.
std::atomic<int> g_partition{0};  // 0 auto, 1 off, 2 force when the layout allows

uint32_t partition_groups(const ph_gpu_index* ix, uint64_t n, int out_width) {
    const int mode = g_partition.load();
    if (mode == 1 || !ix->pool || ix->dev.hot_b < ix->dev.B) return 0;  // needs file order
    const uint64_t pb = ix->info.pilot_bytes;
    // pass B stores non-minimal slots (minimal: remapped) in the output width
    if (out_width == PH_OUT_U32 && ix->info.parts * ix->info.slots_per_part > (uint64_t{1} << 32))
        return 0;
    if (mode == 0 && (pb <= (uint64_t{64} << 20) || n < pb / 32 || ix->dev.window_bytes))
        return 0;
    // pilot bytes per group (L2-resident with pass B's evict_last loads). Fewer, larger
    // groups mean longer runs, i.e. fewer bulk copies and atomics in passes A and C; the
    // sweep at config 3 (profiles/r01_partition_slice_sweep.txt) has its optimum at 32 MiB
    // (G = 11: 10.2 ms; 12 MiB 11.6 ms, 64 MiB 10.6 ms). PH_GPU_PART_SLICE_MB overrides.
    uint64_t slice = uint64_t{32} << 20;
    if (const char* e = std::getenv("PH_GPU_PART_SLICE_MB"))
        if (std::atoll(e) > 0) slice = static_cast<uint64_t>(std::atoll(e)) << 20;
    if (const char* e = std::getenv("PH_GPU_PART_SLICE_KB"))  // (tests: many groups)
        if (std::atoll(e) > 0) slice = static_cast<uint64_t>(std::atoll(e)) << 10;
    uint64_t G = (pb + slice - 1) / slice;
    if (G < 2) G = 2;
    return G > 64 ? 0 : static_cast<uint32_t>(G);
}

// Runs the partitioned path; returns cudaErrorMemoryAllocation (and leaves nothing queued)
// when the scratch cannot be had, so the caller can fall back to the direct kernel.
cudaError_t run_partitioned(const ph_gpu_index* ix, const uint64_t* keys, int src_kind,
                            uint64_t seq_words, uint32_t kbits, void* out, int out_width,
                            uint64_t n, int minimal, uint32_t G, cudaStream_t s) {
    void* scratch = nullptr;
    const uint64_t bytes = phg::partition_scratch_bytes(n, G, out_width);
    if (cudaMallocFromPoolAsync(&scratch, bytes, ix->pool, s) != cudaSuccess) {
        cudaGetLastError();
        return cudaErrorMemoryAllocation;
    }
    const cudaError_t e = phg::launch_query_partitioned(ix->dev, ix->info.bucket_fn, ix->info.pow2,
                                                        keys, src_kind, seq_words, kbits, out,
                                                        out_width, n, minimal, G, scratch, s,
                                                        ix->sms);
    cudaFreeAsync(scratch, s);
    return e;
}

int check_width(int w) {
    return (w == PH_OUT_U32 || w == PH_OUT_U64) ? PH_OK
                                                 : fail(PH_E_INVALID, "out_width must be 4 or 8");
}

int check_u32_range(const ph_gpu_index* ix, int out_width, int minimal) {
    if (out_width == PH_OUT_U64) return PH_OK;
    const uint64_t hi = minimal ? ix->info.n : ix->info.parts * ix->info.slots_per_part;
    if (hi > (uint64_t{1} << 32))
        return fail(PH_E_INVALID, "u32 output cannot hold indices up to " + std::to_string(hi));
    return PH_OK;
}

bool is_device_ptr(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}
bool is_pinned_host(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

}  // namespace

extern "C" {

namespace {
void free_pipelines(ph_gpu_index* ix);  // (with the host-path pipelines below)
}

const char* ph_gpu_last_error(void) { return g_err.c_str(); }
uint64_t ph_gpu_launch_count(void) { return phg::launch_count(); }
int ph_gpu_set_pass_timing(int on) {
    phg::set_pass_timing(on != 0);
    return PH_OK;
}
int ph_gpu_pass_times(double* ms_sums3, int* calls) {
    if (!ms_sums3 || !calls) return fail(PH_E_INVALID, "null argument");
    return phg::pass_times(ms_sums3, calls) == 0 ? PH_OK
                                                 : fail(PH_E_CUDA, "pass timing events failed");
}
int ph_gpu_check_errors(uint64_t* count, uint64_t* first_line) {
    if (!count || !first_line) return fail(PH_E_INVALID, "null argument");
    const int r = phg::check_errors(count, first_line);
    if (r == -1) return fail(PH_E_UNSUPPORTED, "not a checked build (-DPH_CHECKS)");
    return r == 0 ? PH_OK : fail(PH_E_CUDA, "reading the check counters failed");
}
int ph_gpu_set_partition(int mode) {
    if (mode < 0 || mode > 2) return fail(PH_E_INVALID, "partition mode must be 0, 1 or 2");
    g_partition.store(mode);
    return PH_OK;
}
int ph_gpu_set_regime(int regime) {
    if (regime < 0 || regime > 2) return fail(PH_E_INVALID, "regime must be 0..2");
    phg::set_regime(regime);
    return PH_OK;
}
int ph_gpu_set_defer_min(uint64_t min_keys) {
    g_defer_min.store(min_keys);
    return PH_OK;
}
int ph_gpu_set_launch(int threads, int bps) {
    if (threads != 0 && (threads < 32 || threads > 1024 || threads % 32))
        return fail(PH_E_INVALID, "threads_per_block must be a multiple of 32 in [32,1024]");
    phg::set_launch(threads, bps);
    return PH_OK;
}

int ph_gpu_index_create(const uint8_t* ptrh, size_t len, int device, ph_gpu_index** out) {
    PH_RANGE("ph_gpu_index_create");
    if (!out) return fail(PH_E_INVALID, "null out handle");
    *out = nullptr;
    Parsed p;
    if (int rc = parse_ptrh(ptrh, len, p)) return rc;
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0)
        return fail(PH_E_CUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
    if (device < 0 || device >= ndev) return fail(PH_E_INVALID, "bad device ordinal");
    // The kernels use 32-bit P, B, S products. Every shape compute_shape()
    // produces for n < 2^32 satisfies this; larger ones are rejected, not mis-answered.
    if (p.P >= (uint64_t{1} << 32) || p.B >= (uint64_t{1} << 32) || p.S >= (uint64_t{1} << 32))
        return fail(PH_E_UNSUPPORTED, "shape needs P, B, S < 2^32 on the GPU path");
    DeviceGuard g(device);
    if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");

    auto* ix = new ph_gpu_index();
    ix->device = device;
    ix->pl_free = free_pipelines;
    cudaDeviceGetAttribute(&ix->sms, cudaDevAttrMultiProcessorCount, device);
    ph_gpu_info& I = ix->info;
    I.n = p.n;
    I.parts = p.P;
    I.slots_per_part = p.S;
    I.buckets_per_part = p.B;
    I.seed = p.seed;
    I.pilot_bytes = p.pilots_len;
    I.remap_values = p.P * p.S - p.n;
    I.key_kind = p.key_kind;
    I.hash_algo = p.algo;
    I.bucket_fn = p.bucket_fn;
    I.remap_kind = p.remap_kind;
    I.reduce_kind = p.reduce_kind;
    I.pow2 = is_pow2(p.S) ? 1 : 0;
    I.device = device;

    // Default layout: L2-sized pilot arrays keep the file order under a persisting window
    // over all of it; DRAM-sized ones keep the file order without a window, so large
    // device-resident batches take the partitioned path (10.2 ms at config 3
    // against 15.3 ms for the direct kernel on the hot-first layout, which
    // ph_gpu_index_set_l2_policy(index, 64 << 20, 0) selects).
    int rc = p.pilots_len > kDefaultHotBytes
                 ? apply_pilot_layout(ix, p.pilots, 0, kL2NoWindow)
                 : apply_pilot_layout(ix, p.pilots, kDefaultHotBytes, kDefaultL2Flags);
    if (!rc && p.remap_kind != 2) {
        rc = upload(p.remap, p.remap_len, &ix->d_remap);
        I.remap_bytes = p.remap_len;
    }
    if (!rc && p.remap_kind == 2) {
        for (int a = 0; a < 3 && !rc; a++) {
            rc = upload(p.ef[a].data(), p.ef[a].size() * 8, &ix->d_ef[a]);
            I.remap_bytes += p.ef[a].size() * 8;
        }
    }
    if (!rc && p.bucket_fn == 4) {
        std::vector<uint64_t> t;
        optimal_table(t);
        rc = upload(t.data(), t.size() * 8, &ix->d_opt);
    }
    if (!rc && p.key_kind == 1) {
        cudaError_t e = cudaMalloc(&ix->d_aes, 4096);
        if (e == cudaSuccess) e = phg::launch_fill_aes_tab(static_cast<uint32_t*>(ix->d_aes), nullptr);
        if (e == cudaSuccess) e = cudaStreamSynchronize(nullptr);
        if (e != cudaSuccess) rc = cuda_fail(e, "AES table upload");
    }
    if (rc) {
        release(ix);
        return rc;
    }
    phg::DevIndex& d = ix->dev;
    d.aes_tab = static_cast<const uint32_t*>(ix->d_aes);
    d.pilots = static_cast<const uint8_t*>(ix->d_pilots);
    d.remap = static_cast<const uint8_t*>(ix->d_remap);
    d.ef_low = static_cast<const uint64_t*>(ix->d_ef[0]);
    d.ef_high = static_cast<const uint64_t*>(ix->d_ef[1]);
    d.ef_samples = static_cast<const uint64_t*>(ix->d_ef[2]);
    d.opt_table = static_cast<const uint64_t*>(ix->d_opt);
    d.n = p.n;
    d.P = p.P;
    d.S = p.S;
    d.B = p.B;
    d.seed = p.seed;
    if (!I.pow2) {  // FastModU64::make, reduce.hpp:31-36
        const u128 m = ~u128{0} / p.S + 1;
        d.magic_hi = static_cast<uint64_t>(m >> 64);
        d.magic_lo = static_cast<uint64_t>(m);
        d.mod_m64 = static_cast<uint64_t>((u128{1} << 64) / p.S);
        const phg::ModFast mf = phg::mod_fast_make(p.S);  // same remainder, 32-bit products
        d.mod_fast_ok = mf.ok && !std::getenv("PH_GPU_NO_MODFAST");
        d.mod_nS = mf.nS;
        d.mod_c = mf.c;
        d.mod_m1 = mf.m1;
        d.mod_m2 = mf.m2;
    }
    d.hp_base = phg::kC * (p.seed & ~uint64_t{0xff});
    d.seed_lo8 = static_cast<uint32_t>(p.seed & 0xff);
    d.remap_kind = p.remap_kind;
    d.ef_low_bits = p.ef_low_bits;
    d.hash_algo = p.algo;
    {  // AES round keys of hash.cpp:116-119: k0 = (seed^P1, seed+golden), k1 = (mix64(seed)^P2,
       // ~seed*0x6c62272e07bb0143), each (hi, lo) with lo = bytes 0-7
        auto mix64 = [](uint64_t z) {
            z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
            z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
            return z ^ (z >> 31);
        };
        const uint64_t k0hi = p.seed ^ 0x8bb84b93962eacc9ULL, k0lo = p.seed + 0x9e3779b97f4a7c15ULL;
        const uint64_t k1hi = mix64(p.seed) ^ 0x2d358dccaa6c78a5ULL;
        const uint64_t k1lo = (~p.seed) * 0x6c62272e07bb0143ULL;
        const uint64_t w0[2] = {k0lo, k0hi}, w1[2] = {k1lo, k1hi};
        for (int i = 0; i < 4; i++) {
            d.aes_k0[i] = static_cast<uint32_t>(w0[i / 2] >> (32 * (i % 2)));
            d.aes_k1[i] = static_cast<uint32_t>(w1[i / 2] >> (32 * (i % 2)));
        }
    }
    {  // per-index memory pool for per-call scratch (kept cached between calls)
        cudaMemPoolProps props = {};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = device;
        if (cudaMemPoolCreate(&ix->pool, &props) == cudaSuccess) {
            // Freed per-call scratch stays mapped for the next call up to a ceiling of a
            // quarter of the device's memory (a 1e9-key partitioned call takes ~29 GB, and
            // re-mapping it costs ~27 ms per call: measured 37.4 vs 10.2 ms per step with a
            // 2 GiB ceiling); beyond the ceiling it goes back to the device at the caller's
            // next synchronisation. ph_gpu_index_set_scratch_limit changes the ceiling,
            // ph_gpu_index_trim releases everything not in use.
            size_t free_b = 0, total_b = 0;
            cudaMemGetInfo(&free_b, &total_b);
            uint64_t keep = total_b / 4;
            cudaMemPoolSetAttribute(ix->pool, cudaMemPoolAttrReleaseThreshold, &keep);
        } else {
            cudaGetLastError();
            ix->pool = nullptr;  // no deferral: inline remap only
        }
    }
    *out = ix;
    return PH_OK;
}

int ph_gpu_index_destroy(ph_gpu_index* index) {
    release(index);
    return PH_OK;
}

int ph_gpu_index_trim(const ph_gpu_index* index) {
    if (!index) return fail(PH_E_INVALID, "null index");
    if (!index->pool) return PH_OK;
    DeviceGuard g(index->device);
    if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
    const cudaError_t e = cudaMemPoolTrimTo(index->pool, 0);  // only memory not in use
    return e == cudaSuccess ? PH_OK : cuda_fail(e, "cudaMemPoolTrimTo");
}

int ph_gpu_index_set_scratch_limit(ph_gpu_index* index, uint64_t bytes) {
    if (!index) return fail(PH_E_INVALID, "null index");
    if (!index->pool) return PH_OK;
    DeviceGuard g(index->device);
    if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
    const cudaError_t e =
        cudaMemPoolSetAttribute(index->pool, cudaMemPoolAttrReleaseThreshold, &bytes);
    return e == cudaSuccess ? PH_OK : cuda_fail(e, "cudaMemPoolSetAttribute");
}

int ph_gpu_index_set_l2_policy(ph_gpu_index* index, uint64_t hot_bytes, int flags) {
    PH_RANGE("ph_gpu_index_set_l2_policy");
    if (!index) return fail(PH_E_INVALID, "null index");
    DeviceGuard g(index->device);
    if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
    // recover the file-order pilots from the current device layout, then re-lay them out
    const uint64_t P = index->info.parts, B = index->info.buckets_per_part;
    std::vector<uint8_t> cur(P * B), file(P * B);
    PH_CUDA(cudaDeviceSynchronize());
    PH_CUDA(cudaMemcpy(cur.data(), index->d_pilots, cur.size(), cudaMemcpyDeviceToHost));
    const uint64_t H = index->dev.hot_b;
    for (uint64_t part = 0; part < P; part++) {
        std::memcpy(file.data() + part * B, cur.data() + part * H, H);
        std::memcpy(file.data() + part * B + H, cur.data() + P * H + part * (B - H), B - H);
    }
    return apply_pilot_layout(index, file.data(), hot_bytes, flags);  // swaps only on success
}

int ph_gpu_index_info(const ph_gpu_index* index, ph_gpu_info* out) {
    if (!index || !out) return fail(PH_E_INVALID, "null argument");
    *out = index->info;
    return PH_OK;
}

int ph_gpu_query_u64(const ph_gpu_index* ix, const uint64_t* d_keys, size_t n, void* d_out,
                     int out_width, int minimal, ph_gpu_stream_t stream) {
    PH_RANGE("ph_gpu_query_u64");
    if (!ix) return fail(PH_E_INVALID, "null index");
    if (ix->info.key_kind != 0) return fail(PH_E_KEYKIND, "u64 query on a string-key index");
    if (int rc = check_width(out_width)) return rc;
    if (int rc = check_u32_range(ix, out_width, minimal)) return rc;
    if (n == 0) return PH_OK;
    if (!d_keys || !d_out) return fail(PH_E_INVALID, "null key or output pointer");
    if ((reinterpret_cast<uintptr_t>(d_keys) & 7) || (reinterpret_cast<uintptr_t>(d_out) & (out_width - 1)))
        return fail(PH_E_INVALID, "keys must be 8-byte aligned and out aligned to out_width");
    DeviceGuard g(ix->device);
    if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
    if (const uint32_t G = partition_groups(ix, n, out_width)) {
        const cudaError_t pe = run_partitioned(ix, d_keys, 0, 0, 0, d_out, out_width, n, minimal,
                                               G, static_cast<cudaStream_t>(stream));
        if (pe != cudaErrorMemoryAllocation)
            return pe == cudaSuccess ? PH_OK : cuda_fail(pe, "query_u64 (partitioned)");
    }
    DeferScratch ds(ix, n, minimal, static_cast<cudaStream_t>(stream));
    cudaError_t e = phg::launch_query_u64(ix->dev, ix->info.bucket_fn, ix->info.pow2, d_keys, d_out,
                                          out_width, n, minimal, static_cast<cudaStream_t>(stream),
                                          ix->sms, ds.rl);
    return e == cudaSuccess ? PH_OK : cuda_fail(e, "query_u64 launch");
}

int ph_gpu_query_bytes(const ph_gpu_index* ix, const uint8_t* d_bytes, const uint64_t* d_offsets,
                       size_t n, void* d_out, int out_width, int minimal,
                       ph_gpu_stream_t stream) {
    PH_RANGE("ph_gpu_query_bytes");
    if (!ix) return fail(PH_E_INVALID, "null index");
    if (ix->info.key_kind != 1) return fail(PH_E_KEYKIND, "string query on a u64-key index");
    if (int rc = check_width(out_width)) return rc;
    if (int rc = check_u32_range(ix, out_width, minimal)) return rc;
    if (n == 0) return PH_OK;
    if (!d_bytes || !d_offsets || !d_out) return fail(PH_E_INVALID, "null pointer argument");
    if ((reinterpret_cast<uintptr_t>(d_offsets) & 7) || (reinterpret_cast<uintptr_t>(d_out) & (out_width - 1)))
        return fail(PH_E_INVALID, "offsets must be 8-byte aligned and out aligned to out_width");
    DeviceGuard g(ix->device);
    if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
    cudaError_t e = phg::launch_query_bytes(ix->dev, ix->info.bucket_fn, ix->info.pow2, d_bytes,
                                            d_offsets, 0, d_out, out_width, n, minimal,
                                            static_cast<cudaStream_t>(stream), ix->sms);
    return e == cudaSuccess ? PH_OK : cuda_fail(e, "query_bytes launch");
}

// ---------------------------------------------------------------------------
// host-resident bulk queries: chunked pipeline over kSlots streams
// ---------------------------------------------------------------------------
namespace {

constexpr int kSlots = 3;

struct Slot {
    cudaStream_t s = nullptr;
    void* d_in = nullptr;   // keys (u64) or bytes
    void* d_off = nullptr;  // offsets (bytes path)
    void* d_out = nullptr;
    void* h_in = nullptr;   // pinned bounce buffers (pageable callers only)
    void* h_off = nullptr;
    void* h_out = nullptr;
    size_t pend_off = 0, pend_n = 0;  // chunk whose output still sits in h_out
    bool pending = false;
};

struct Pipeline {
    Slot slot[kSlots];
    size_t in_bytes = 0, off_bytes = 0, out_bytes = 0;
    bool bounce = false;
    ~Pipeline() {
        for (Slot& s : slot) {
            if (s.s) cudaStreamSynchronize(s.s);
            cudaFree(s.d_in);
            cudaFree(s.d_off);
            cudaFree(s.d_out);
            cudaFreeHost(s.h_in);
            cudaFreeHost(s.h_off);
            cudaFreeHost(s.h_out);
            if (s.s) cudaStreamDestroy(s.s);
        }
    }
};

int alloc_pipeline(Pipeline& pl, size_t in_bytes, size_t off_bytes, size_t out_bytes,
                   bool bounce) {
    pl.in_bytes = in_bytes;
    pl.off_bytes = off_bytes;
    pl.out_bytes = out_bytes;
    pl.bounce = bounce;
    for (Slot& s : pl.slot) {
        PH_CUDA(cudaStreamCreateWithFlags(&s.s, cudaStreamNonBlocking));
        if (cudaMalloc(&s.d_in, in_bytes ? in_bytes : 1) != cudaSuccess ||
            (off_bytes && cudaMalloc(&s.d_off, off_bytes) != cudaSuccess) ||
            cudaMalloc(&s.d_out, out_bytes) != cudaSuccess)
            return fail(PH_E_NOMEM, "device staging allocation failed");
        if (bounce) {
            if (cudaHostAlloc(&s.h_in, in_bytes ? in_bytes : 1, 0) != cudaSuccess ||
                (off_bytes && cudaHostAlloc(&s.h_off, off_bytes, 0) != cudaSuccess) ||
                cudaHostAlloc(&s.h_out, out_bytes, 0) != cudaSuccess)
                return fail(PH_E_NOMEM, "pinned staging allocation failed");
        }
    }
    return PH_OK;
}

// A pipeline borrowed from the index's cache for one host-path call (allocating streams
// and staging buffers per call cost up to hundreds of ms when cudaFree synchronised the
// device); concurrent callers get separate pipelines.
struct PipelineLease {
    const ph_gpu_index* ix = nullptr;
    Pipeline* p = nullptr;
    ~PipelineLease() {
        if (!p) return;
        for (Slot& s : p->slot)
            if (s.s) cudaStreamSynchronize(s.s);
        std::lock_guard<std::mutex> lk(ix->pl_mu);
        if (ix->pl_cache.size() < 4) {
            for (Slot& s : p->slot) s.pending = false;
            ix->pl_cache.push_back(p);
        } else {
            delete p;
        }
    }
    Pipeline& operator*() { return *p; }
};

void free_pipelines(ph_gpu_index* ix);

int lease_pipeline(const ph_gpu_index* ix, size_t in_bytes, size_t off_bytes, size_t out_bytes,
                   bool bounce, PipelineLease& L) {
    L.ix = ix;
    {
        std::lock_guard<std::mutex> lk(ix->pl_mu);
        for (size_t i = 0; i < ix->pl_cache.size(); i++) {
            Pipeline* c = ix->pl_cache[i];
            if (c->bounce == bounce && c->in_bytes >= in_bytes && c->off_bytes >= off_bytes &&
                c->out_bytes >= out_bytes) {
                ix->pl_cache.erase(ix->pl_cache.begin() + static_cast<long>(i));
                L.p = c;
                return PH_OK;
            }
        }
    }
    auto* p = new Pipeline();
    if (int rc = alloc_pipeline(*p, in_bytes, off_bytes, out_bytes, bounce)) {
        delete p;
        return rc;
    }
    L.p = p;
    return PH_OK;
}

void free_pipelines(ph_gpu_index* ix) {
    std::lock_guard<std::mutex> lk(ix->pl_mu);
    for (Pipeline* p : ix->pl_cache) delete p;
    ix->pl_cache.clear();
}

// Keys per pipeline chunk (default 8 Mi = 64 MiB of u64 keys); PH_GPU_CHUNK_KEYS overrides
// (tools/e2e_sweep.py).
size_t chunk_keys(size_t n) {
    size_t c = size_t{1} << 23;
    if (const char* e = std::getenv("PH_GPU_CHUNK_KEYS")) {
        const unsigned long long v = std::strtoull(e, nullptr, 10);
        if (v >= 1024) c = static_cast<size_t>(v) & ~size_t{31};
    }
    return n < c ? n : c;
}

}  // namespace

int ph_gpu_index_stream_u64(const ph_gpu_index* ix, const uint64_t* h_keys, size_t n, void* h_out,
                            int out_width, int minimal) {
    PH_RANGE("ph_gpu_index_stream_u64");
    if (!ix) return fail(PH_E_INVALID, "null index");
    if (ix->info.key_kind != 0) return fail(PH_E_KEYKIND, "u64 query on a string-key index");
    if (int rc = check_width(out_width)) return rc;
    if (int rc = check_u32_range(ix, out_width, minimal)) return rc;
    if (n == 0) return PH_OK;
    if (!h_keys || !h_out) return fail(PH_E_INVALID, "null key or output pointer");
    DeviceGuard g(ix->device);
    if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
    {
        const bool dk = is_device_ptr(h_keys), dout = is_device_ptr(h_out);
        if (dk != dout) return fail(PH_E_INVALID, "keys and out must both be host or both device memory");
        if (dk) {  // device spans: no staging
            if (int rc = ph_gpu_query_u64(ix, h_keys, n, h_out, out_width, minimal, nullptr)) return rc;
            PH_CUDA(cudaStreamSynchronize(nullptr));
            return PH_OK;
        }
    }
    const size_t C = chunk_keys(n);
    const bool bounce = !(is_pinned_host(h_keys) && is_pinned_host(h_out));
    PipelineLease lease;
    if (int rc = lease_pipeline(ix, C * 8, 0, C * out_width, bounce, lease)) return rc;
    Pipeline& pl = *lease;
    auto* out_b = static_cast<uint8_t*>(h_out);
    auto drain = [&](Slot& s) -> int {
        if (!s.pending) return PH_OK;
        PH_CUDA(cudaStreamSynchronize(s.s));
        std::memcpy(out_b + s.pend_off * out_width, s.h_out, s.pend_n * out_width);
        s.pending = false;
        return PH_OK;
    };
    size_t c = 0;
    for (size_t off = 0; off < n; off += C, c++) {
        Slot& s = pl.slot[c % kSlots];
        const size_t m = n - off < C ? n - off : C;
        const void* src = h_keys + off;
        void* dst = out_b + off * out_width;
        if (bounce) {
            if (int rc = drain(s)) return rc;
            std::memcpy(s.h_in, h_keys + off, m * 8);
            src = s.h_in;
            dst = s.h_out;
        }
        PH_CUDA(cudaMemcpyAsync(s.d_in, src, m * 8, cudaMemcpyHostToDevice, s.s));
        {
            DeferScratch ds(ix, m, minimal, s.s);
            PH_CUDA(phg::launch_query_u64(ix->dev, ix->info.bucket_fn, ix->info.pow2,
                                          static_cast<const uint64_t*>(s.d_in), s.d_out, out_width,
                                          m, minimal, s.s, ix->sms, ds.rl));
        }
        PH_CUDA(cudaMemcpyAsync(dst, s.d_out, m * out_width, cudaMemcpyDeviceToHost, s.s));
        if (bounce) {
            s.pending = true;
            s.pend_off = off;
            s.pend_n = m;
        }
    }
    for (Slot& s : pl.slot) {
        if (bounce) {
            if (int rc = drain(s)) return rc;
        } else {
            PH_CUDA(cudaStreamSynchronize(s.s));
        }
    }
    return PH_OK;
}

int ph_gpu_index_stream_bytes(const ph_gpu_index* ix, const uint8_t* h_bytes,
                              const uint64_t* h_offsets, size_t n, void* h_out, int out_width,
                              int minimal) {
    PH_RANGE("ph_gpu_index_stream_bytes");
    if (!ix) return fail(PH_E_INVALID, "null index");
    if (ix->info.key_kind != 1) return fail(PH_E_KEYKIND, "string query on a u64-key index");
    if (int rc = check_width(out_width)) return rc;
    if (int rc = check_u32_range(ix, out_width, minimal)) return rc;
    if (n == 0) return PH_OK;
    if (!h_bytes || !h_offsets || !h_out) return fail(PH_E_INVALID, "null pointer argument");
    DeviceGuard g(ix->device);
    if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
    {
        const bool db = is_device_ptr(h_bytes), doff = is_device_ptr(h_offsets),
                   dout = is_device_ptr(h_out);
        if (db != doff || db != dout)
            return fail(PH_E_INVALID, "bytes, offsets and out must all be host or all device memory");
        if (db) {  // device spans: no staging
            if (int rc = ph_gpu_query_bytes(ix, h_bytes, h_offsets, n, h_out, out_width, minimal,
                                            nullptr))
                return rc;
            PH_CUDA(cudaStreamSynchronize(nullptr));
            return PH_OK;
        }
    }
    const size_t C = chunk_keys(n);
    size_t max_bytes = 0;
    for (size_t off = 0; off < n; off += C) {
        const size_t m = n - off < C ? n - off : C;
        const size_t b = h_offsets[off + m] - h_offsets[off];
        if (b > max_bytes) max_bytes = b;
    }
    const bool bounce = !(is_pinned_host(h_bytes) && is_pinned_host(h_offsets) &&
                          is_pinned_host(h_out));
    PipelineLease lease;
    if (int rc = lease_pipeline(ix, max_bytes, (C + 1) * 8, C * out_width, bounce, lease))
        return rc;
    Pipeline& pl = *lease;
    auto* out_b = static_cast<uint8_t*>(h_out);
    auto drain = [&](Slot& s) -> int {
        if (!s.pending) return PH_OK;
        PH_CUDA(cudaStreamSynchronize(s.s));
        std::memcpy(out_b + s.pend_off * out_width, s.h_out, s.pend_n * out_width);
        s.pending = false;
        return PH_OK;
    };
    size_t c = 0;
    for (size_t off = 0; off < n; off += C, c++) {
        Slot& s = pl.slot[c % kSlots];
        const size_t m = n - off < C ? n - off : C;
        const uint64_t b0 = h_offsets[off], b1 = h_offsets[off + m];
        const void* src_b = h_bytes + b0;
        const void* src_o = h_offsets + off;
        void* dst = out_b + off * out_width;
        if (bounce) {
            if (int rc = drain(s)) return rc;
            std::memcpy(s.h_in, h_bytes + b0, b1 - b0);
            std::memcpy(s.h_off, h_offsets + off, (m + 1) * 8);
            src_b = s.h_in;
            src_o = s.h_off;
            dst = s.h_out;
        }
        if (b1 > b0) PH_CUDA(cudaMemcpyAsync(s.d_in, src_b, b1 - b0, cudaMemcpyHostToDevice, s.s));
        PH_CUDA(cudaMemcpyAsync(s.d_off, src_o, (m + 1) * 8, cudaMemcpyHostToDevice, s.s));
        PH_CUDA(phg::launch_query_bytes(ix->dev, ix->info.bucket_fn, ix->info.pow2,
                                        static_cast<const uint8_t*>(s.d_in),
                                        static_cast<const uint64_t*>(s.d_off), b0, s.d_out,
                                        out_width, m, minimal, s.s, ix->sms));
        PH_CUDA(cudaMemcpyAsync(dst, s.d_out, m * out_width, cudaMemcpyDeviceToHost, s.s));
        if (bounce) {
            s.pending = true;
            s.pend_off = off;
            s.pend_n = m;
        }
    }
    for (Slot& s : pl.slot) {
        if (bounce) {
            if (int rc = drain(s)) return rc;
        } else {
            PH_CUDA(cudaStreamSynchronize(s.s));
        }
    }
    return PH_OK;
}

int ph_gpu_query_kmers(const ph_gpu_index* ix, const uint64_t* d_seq, uint64_t n_bases, int k,
                       void* d_out, int out_width, int minimal, ph_gpu_stream_t stream) {
    PH_RANGE("ph_gpu_query_kmers");
    if (!ix) return fail(PH_E_INVALID, "null index");
    if (ix->info.key_kind != 0) return fail(PH_E_KEYKIND, "k-mer query on a string-key index");
    if (k < 1 || k > 32) return fail(PH_E_INVALID, "k must be in [1, 32]");
    if (int rc = check_width(out_width)) return rc;
    if (int rc = check_u32_range(ix, out_width, minimal)) return rc;
    if (n_bases < (uint64_t)k) return PH_OK;
    if (!d_seq || !d_out) return fail(PH_E_INVALID, "null sequence or output pointer");
    if ((reinterpret_cast<uintptr_t>(d_seq) & 7) || (reinterpret_cast<uintptr_t>(d_out) & (out_width - 1)))
        return fail(PH_E_INVALID, "seq must be 8-byte aligned and out aligned to out_width");
    DeviceGuard g(ix->device);
    if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
    const uint64_t nwin = n_bases - (uint64_t)k + 1;
    if (const uint32_t G = partition_groups(ix, nwin, out_width)) {
        const cudaError_t pe = run_partitioned(ix, d_seq, 1, (n_bases + 31) / 32, (uint32_t)(2 * k),
                                               d_out, out_width, nwin, minimal, G,
                                               static_cast<cudaStream_t>(stream));
        if (pe != cudaErrorMemoryAllocation)
            return pe == cudaSuccess ? PH_OK : cuda_fail(pe, "query_kmers (partitioned)");
    }
    DeferScratch ds(ix, nwin, minimal, static_cast<cudaStream_t>(stream));
    cudaError_t e = phg::launch_query_kmers(ix->dev, ix->info.bucket_fn, ix->info.pow2, d_seq,
                                            n_bases, k, d_out, out_width, minimal,
                                            static_cast<cudaStream_t>(stream), ix->sms, ds.rl);
    return e == cudaSuccess ? PH_OK : cuda_fail(e, "query_kmers launch");
}

int ph_gpu_index_stream_kmers(const ph_gpu_index* ix, const uint64_t* h_seq, uint64_t n_bases,
                              int k, void* h_out, int out_width, int minimal) {
    PH_RANGE("ph_gpu_index_stream_kmers");
    if (!ix) return fail(PH_E_INVALID, "null index");
    if (ix->info.key_kind != 0) return fail(PH_E_KEYKIND, "k-mer query on a string-key index");
    if (k < 1 || k > 32) return fail(PH_E_INVALID, "k must be in [1, 32]");
    if (int rc = check_width(out_width)) return rc;
    if (int rc = check_u32_range(ix, out_width, minimal)) return rc;
    if (n_bases < (uint64_t)k) return PH_OK;
    if (!h_seq || !h_out) return fail(PH_E_INVALID, "null sequence or output pointer");
    DeviceGuard g(ix->device);
    if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
    {
        const bool ds = is_device_ptr(h_seq), dout = is_device_ptr(h_out);
        if (ds != dout) return fail(PH_E_INVALID, "seq and out must both be host or both device memory");
        if (ds) {  // device spans: no staging
            if (int rc = ph_gpu_query_kmers(ix, h_seq, n_bases, k, h_out, out_width, minimal, nullptr))
                return rc;
            PH_CUDA(cudaStreamSynchronize(nullptr));
            return PH_OK;
        }
    }
    const uint64_t n = n_bases - (uint64_t)k + 1;  // windows
    const uint64_t nwords_total = (n_bases + 31) / 32;
    const size_t C = chunk_keys(n) & ~size_t{31} ? chunk_keys(n) & ~size_t{31} : 32;  // windows
    const size_t max_words = (C + (size_t)k - 1 + 31) / 32 + 1;
    const bool bounce = !(is_pinned_host(h_seq) && is_pinned_host(h_out));
    PipelineLease lease;
    if (int rc = lease_pipeline(ix, max_words * 8, 0, C * out_width, bounce, lease)) return rc;
    Pipeline& pl = *lease;
    auto* out_b = static_cast<uint8_t*>(h_out);
    auto drain = [&](Slot& s) -> int {
        if (!s.pending) return PH_OK;
        PH_CUDA(cudaStreamSynchronize(s.s));
        std::memcpy(out_b + s.pend_off * out_width, s.h_out, s.pend_n * out_width);
        s.pending = false;
        return PH_OK;
    };
    size_t c = 0;
    for (uint64_t off = 0; off < n; off += C, c++) {  // off is a multiple of 32
        Slot& s = pl.slot[c % kSlots];
        const uint64_t m = n - off < C ? n - off : C;
        const uint64_t nb = m + (uint64_t)k - 1;  // bases this chunk reads
        const uint64_t w0 = off / 32;
        uint64_t nw = (nb + 31) / 32;
        if (w0 + nw > nwords_total) nw = nwords_total - w0;
        const void* src = h_seq + w0;
        void* dst = out_b + off * out_width;
        if (bounce) {
            if (int rc = drain(s)) return rc;
            std::memcpy(s.h_in, h_seq + w0, nw * 8);
            src = s.h_in;
            dst = s.h_out;
        }
        PH_CUDA(cudaMemcpyAsync(s.d_in, src, nw * 8, cudaMemcpyHostToDevice, s.s));
        {
            DeferScratch ds(ix, m, minimal, s.s);
            PH_CUDA(phg::launch_query_kmers(ix->dev, ix->info.bucket_fn, ix->info.pow2,
                                            static_cast<const uint64_t*>(s.d_in), nb, k, s.d_out,
                                            out_width, minimal, s.s, ix->sms, ds.rl));
        }
        PH_CUDA(cudaMemcpyAsync(dst, s.d_out, m * out_width, cudaMemcpyDeviceToHost, s.s));
        if (bounce) {
            s.pending = true;
            s.pend_off = off;
            s.pend_n = m;
        }
    }
    for (Slot& s : pl.slot) {
        if (bounce) {
            if (int rc = drain(s)) return rc;
        } else {
            PH_CUDA(cudaStreamSynchronize(s.s));
        }
    }
    return PH_OK;
}

// Single-key queries (index.hpp:60-64), synchronous: one kernel launch takes the key as a
// launch parameter (string keys up to 256 bytes; longer ones are written into the index's mapped
// pinned block) and writes the answer into that block, and the call waits on the index's
// single-key stream. Many host threads may call at once; they take turns on the block.
int ph_gpu_index_u64(const ph_gpu_index* ix, uint64_t key, int minimal, uint64_t* out) {
    PH_RANGE("ph_gpu_index_u64");
    if (!ix || !out) return fail(PH_E_INVALID, "null argument");
    if (ix->info.key_kind != 0) return fail(PH_E_KEYKIND, "u64 query on a string-key index");
    DeviceGuard g(ix->device);
    if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
    std::lock_guard<std::mutex> lk(ix->single_mu);
    if (int rc = ensure_single(ix, 0)) return rc;
    auto* h = reinterpret_cast<volatile uint64_t*>(ix->single_h);
    auto* d = reinterpret_cast<uint64_t*>(ix->single_d);
    cudaError_t e = phg::launch_index_u64_one(ix->dev, ix->info.bucket_fn, ix->info.pow2, key,
                                              d + 2, minimal, ix->single_s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ix->single_s);
    if (e != cudaSuccess) return cuda_fail(e, "index_u64");
    *out = h[2];
    return PH_OK;
}

int ph_gpu_index_bytes(const ph_gpu_index* ix, const uint8_t* key, size_t len, int minimal,
                       uint64_t* out) {
    PH_RANGE("ph_gpu_index_bytes");
    if (!ix || !out || (!key && len)) return fail(PH_E_INVALID, "null argument");
    if (ix->info.key_kind != 1) return fail(PH_E_KEYKIND, "string query on a u64-key index");
    DeviceGuard g(ix->device);
    if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
    std::lock_guard<std::mutex> lk(ix->single_mu);
    if (int rc = ensure_single(ix, len <= 256 ? 0 : len)) return rc;
    auto* h = reinterpret_cast<volatile uint64_t*>(ix->single_h);
    auto* d = reinterpret_cast<uint64_t*>(ix->single_d);
    if (len <= 256) {  // the key rides in the launch parameters: no host read by the kernel
        cudaError_t e = phg::launch_index_bytes_one(ix->dev, ix->info.bucket_fn, ix->info.pow2,
                                                    key, static_cast<uint32_t>(len), d + 2,
                                                    minimal, ix->single_s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(ix->single_s);
        if (e != cudaSuccess) return cuda_fail(e, "index_bytes");
        *out = h[2];
        return PH_OK;
    }
    h[0] = 0;  // offsets {0, len}; the bytes follow the header
    h[1] = len;
    if (len) std::memcpy(ix->single_h + kSingleHeader, key, len);
    cudaError_t e = phg::launch_query_bytes(ix->dev, ix->info.bucket_fn, ix->info.pow2,
                                            ix->single_d + kSingleHeader, d, 0, d + 2, 8, 1,
                                            minimal, ix->single_s, ix->sms);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ix->single_s);
    if (e != cudaSuccess) return cuda_fail(e, "index_bytes");
    *out = h[2];
    return PH_OK;
}

// load_index (serde.cpp:251-260) for the GPU: the PTRH file is mmap'ed, pinned in place
// (cudaHostRegister, read-only) so the upload runs at PCIe speed, then validated and
// uploaded exactly as ph_gpu_index_create does.
int ph_gpu_index_load(const char* path, int device, ph_gpu_index** out) {
    PH_RANGE("ph_gpu_index_load");
    if (!path || !out) return fail(PH_E_INVALID, "null argument");
    *out = nullptr;
    const int fd = open(path, O_RDONLY);
    if (fd < 0) return fail(PH_E_INVALID, std::string("cannot open ") + path);
    struct stat st;
    if (fstat(fd, &st) != 0 || st.st_size <= 0) {
        close(fd);
        return fail(PH_E_FORMAT, std::string("index file truncated: ") + path);
    }
    const size_t len = static_cast<size_t>(st.st_size);
    void* m = mmap(nullptr, len, PROT_READ, MAP_PRIVATE | MAP_POPULATE, fd, 0);
    close(fd);
    if (m == MAP_FAILED) return fail(PH_E_INVALID, std::string("mmap failed: ") + path);
    const bool pinned =
        cudaHostRegister(m, len, cudaHostRegisterReadOnly | cudaHostRegisterPortable) == cudaSuccess;
    if (!pinned) cudaGetLastError();  // pageable upload still works
    const int rc = ph_gpu_index_create(static_cast<const uint8_t*>(m), len, device, out);
    if (pinned) cudaHostUnregister(m);
    munmap(m, len);
    return rc;
}

// verify_bijection (proj/tools/ptrhash.cpp:186-210) on the device, synchronous: counts
// outputs >= n and repeated outputs among d_out[0..count).
int ph_gpu_verify_bijection(const void* d_out, size_t count, int out_width, uint64_t n,
                            int device, uint64_t* out_of_range, uint64_t* duplicates) {
    PH_RANGE("ph_gpu_verify_bijection");
    if (!d_out || !out_of_range || !duplicates) return fail(PH_E_INVALID, "null argument");
    if (int rc = check_width(out_width)) return rc;
    DeviceGuard g(device);
    if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    const size_t words = (n + 31) / 32;
    void* scratch = nullptr;
    if (cudaMalloc(&scratch, 16 + words * 4) != cudaSuccess)
        return fail(PH_E_NOMEM, "cudaMalloc(bijection bitset)");
    auto* bad = static_cast<unsigned long long*>(scratch);
    auto* bits = reinterpret_cast<unsigned int*>(static_cast<uint8_t*>(scratch) + 16);
    cudaError_t e = cudaMemset(scratch, 0, 16 + words * 4);
    if (e == cudaSuccess) e = phg::launch_verify(d_out, out_width, count, n, bits, bad, nullptr, sms);
    unsigned long long h[2] = {0, 0};
    if (e == cudaSuccess) e = cudaMemcpy(h, bad, 16, cudaMemcpyDeviceToHost);
    cudaFree(scratch);
    if (e != cudaSuccess) return cuda_fail(e, "verify_bijection");
    *out_of_range = h[0];
    *duplicates = h[1];
    return PH_OK;
}

int ph_gpu_build_prepare_u64(const uint64_t* d_keys, size_t n, uint64_t parts,
                             uint64_t slots_per_part, uint64_t seed, int device,
                             uint64_t* d_hashes, uint64_t* d_offsets, int* status) {
    PH_RANGE("ph_gpu_build_prepare_u64");
    if ((!d_keys && n) || (!d_hashes && n) || !d_offsets || !status)
        return fail(PH_E_INVALID, "null argument");
    if (parts == 0 || slots_per_part == 0) return fail(PH_E_INVALID, "degenerate shape");
    DeviceGuard g(device);
    if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    const cudaError_t e = phg::build_prepare_u64(d_keys, n, parts, slots_per_part, seed, d_hashes,
                                                 d_offsets, status, nullptr, sms);
    return e == cudaSuccess ? PH_OK : cuda_fail(e, "build_prepare_u64");
}

int ph_gpu_bucket_sizes(const ph_gpu_index* index, const uint64_t* d_keys, size_t n,
                        uint64_t* hist, size_t cap, size_t* len) {
    PH_RANGE("ph_gpu_bucket_sizes");
    if (!index || (!d_keys && n) || !len || (!hist && cap)) return fail(PH_E_INVALID, "null argument");
    if (index->info.key_kind != 0) return fail(PH_E_KEYKIND, "index was built over byte-string keys");
    DeviceGuard g(index->device);
    if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
    uint64_t l = 0;
    const cudaError_t e = phg::bucket_size_hist(index->dev, index->info.bucket_fn, d_keys, n, hist,
                                                cap, &l, nullptr, index->sms);
    if (e == cudaErrorNotSupported) return fail(PH_E_UNSUPPORTED, "a bucket holds more than 2^24 keys");
    if (e != cudaSuccess) return cuda_fail(e, "bucket_sizes");
    *len = l;
    return PH_OK;
}

int ph_gpu_gather_replay_u64(const ph_gpu_index* index, const uint64_t* d_keys, size_t n,
                             ph_gpu_stream_t stream) {
    PH_RANGE("ph_gpu_gather_replay_u64");
    if (!index || (!d_keys && n)) return fail(PH_E_INVALID, "null argument");
    if (index->info.key_kind != 0) return fail(PH_E_KEYKIND, "index was built over byte-string keys");
    DeviceGuard g(index->device);
    if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    void* sink = nullptr;
    cudaError_t e = index->pool ? cudaMallocFromPoolAsync(&sink, 256, index->pool, s)
                                : cudaMallocAsync(&sink, 256, s);
    if (e != cudaSuccess) return cuda_fail(e, "gather_replay scratch");
    e = phg::launch_gather_replay(index->dev, index->info.bucket_fn, d_keys, n,
                                  static_cast<uint32_t*>(sink), s, index->sms);
    cudaFreeAsync(sink, s);
    return e == cudaSuccess ? PH_OK : cuda_fail(e, "gather_replay");
}

}  // extern "C"
