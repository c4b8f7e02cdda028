// ph_builder.cu — construction of a PTRH v1 index over u64 keys with the data-parallel
// front of each build attempt on the GPU. Off the query path.
//
// One attempt of the reference's build (construction.cpp:28-60, run_attempt) is
//   hash_all + scatter_to_parts + per-part sort   -> GPU: phg::build_prepare_u64
//                                                    (hash fused into a hand-written MSD
//                                                    radix sort, ph_sort.cu; part offsets)
//   build_parts: per part, the hash-and-displace   -> host threads, one part at a time,
//     pilot search (engine.hpp:105-292)               fed part by part from the device
//                                                     through a ring of pinned buffers
//   assemble_remap (engine.hpp:544-557)             -> host
// and the attempt loop reseeds exactly as build_u64_impl (construction.cpp:113-138). The
// output is the same PTRH byte string the reference's build() + serialize() produce for the
// same keys and parameters (tests/test_builder.py checks this against the reference).
//
// The pilot search is sequential within a part by definition (the greedy order and the
// eviction choices decide the pilots), so it stays on the CPU as the survey plans; parts
// run in parallel. Everything here is restated from the reference's documented algorithm
// with our own data structures: the priority queue is the bucket list pre-sorted by
// (size desc, id asc) merged with a heap of evicted buckets, the slot reduction is an exact
// y mod S, and hash_pilot is a 256-entry table.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <queue>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/ph_gpu.h"
#include "ph_kernels.h"
#include "ph_nvtx.h"

namespace phg {
int report_error(int code, const std::string& msg);  // ph_abi.cu (thread-local last error)
void optimal_gamma_table(std::vector<uint64_t>& t);  // ph_abi.cu (bucket_fn.cpp:16-39)
}  // namespace phg

namespace {

using u128 = unsigned __int128;
constexpr uint64_t kMix = 0x517cc1b727220a95ULL;     // hash.hpp:13
constexpr uint64_t kGolden = 0x9e3779b97f4a7c15ULL;  // common.hpp:60
constexpr uint32_t kNone = UINT32_MAX;               // engine.hpp:91 (no bucket)
constexpr int kRecent = 16;                          // engine.hpp:92

struct BuildFail : std::runtime_error {
    int code;
    BuildFail(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

inline uint64_t mulhi(uint64_t a, uint64_t b) { return (uint64_t)(((u128)a * b) >> 64); }
inline bool pow2(uint64_t x) { return x && !(x & (x - 1)); }
inline uint64_t ceil_div128(u128 a, u128 b) { return (uint64_t)((a + b - 1) / b); }

// ---- parameters and shape (shape.hpp:46-97, shape.cpp:52-145) ---------------------------

void validate(const ph_build_params& p) {
    if (!p.alpha_num || !p.alpha_den || p.alpha_num > p.alpha_den)
        throw BuildFail(PH_E_INVALID, "alpha must be in (0, 1]");
    if (!p.lambda_den || p.lambda_num < p.lambda_den)
        throw BuildFail(PH_E_INVALID, "lambda must be >= 1");
    if (p.bucket_fn > 4 || p.remap_kind > 2 || p.reduce_kind > 2)
        throw BuildFail(PH_E_INVALID, "unknown bucket function, remap kind or reduce kind");
    if (p.remap_kind == 1 && (uint64_t)p.alpha_num * 100 > (uint64_t)p.alpha_den * 99)
        throw BuildFail(PH_E_INVALID, "CacheLineEF remap requires alpha <= 0.99");
}

uint64_t target_keys_per_part(uint64_t n, uint32_t an, uint32_t ad) {
    if (an == ad) return n;  // no slack: one part
    // minimum part size 2/eps^2 with eps = (1-alpha)/2, grown by ln(n/m) (shape.cpp:86-97)
    const double den = ad, gap = (double)(ad - an);
    const double m = 8.0 * den * den / (gap * gap);
    if ((double)n <= m) return (uint64_t)std::ceil(m);
    return (uint64_t)std::ceil(std::max(m, m * std::log((double)n / m)));
}

struct Shape {
    uint64_t n, P, S, B;
};

Shape make_shape(uint64_t n, const ph_build_params& p) {
    Shape s{n, 0, 0, 0};
    const uint64_t an = p.alpha_num, ad = p.alpha_den;
    if (p.reduce_kind == 0) {  // power-of-two S
        const uint64_t kpp = target_keys_per_part(n, p.alpha_num, p.alpha_den);
        uint64_t S = ceil_div128((u128)kpp * ad, an);
        uint64_t c = 1;
        while (c < S) c <<= 1;
        s.S = c;
        s.P = ceil_div128((u128)n * ad, (u128)an * s.S);
    } else if (p.reduce_kind == 1) {  // one part
        uint64_t S = ceil_div128((u128)n * ad, an);
        while (pow2(S)) S++;
        if (S >= (uint64_t{1} << 32)) throw BuildFail(PH_E_INVALID, "single-part mode needs n/alpha < 2^32");
        s.P = 1;
        s.S = S;
    } else {  // several parts, S not a power of two
        const uint64_t kpp = target_keys_per_part(n, p.alpha_num, p.alpha_den);
        const uint64_t P = (n + kpp - 1) / kpp;
        uint64_t S = ceil_div128((u128)n * ad, (u128)an * P);
        if (pow2(S)) S++;
        if (S >= (uint64_t{1} << 32)) throw BuildFail(PH_E_INVALID, "fastmod reduce needs slots per part < 2^32");
        s.P = P;
        s.S = S;
    }
    s.B = ceil_div128((u128)an * s.S * p.lambda_den, (u128)ad * p.lambda_num);
    if (s.P > (uint64_t{1} << 40) || (u128)s.P * s.S > ((u128)1 << 62) ||
        (u128)s.P * s.B > ((u128)1 << 62))
        throw BuildFail(PH_E_INVALID, "shape: slot index range overflow");
    return s;
}

// ---- per-key arithmetic (bucket_fn.hpp:18-78, reduce.hpp:27-77, hash.hpp:27-32) ---------

struct Arith {
    Shape sh;
    int fn;
    const uint64_t* opt;  // optimal-gamma table (65537 entries) or null
    bool p2;
    uint64_t fm;  // floor((2^64-1)/S) for the exact y mod S

    uint64_t gamma(uint64_t x) const {
        switch (fn) {
            case 0: return x;
            case 1: return mulhi(x, x);
            case 2: {
                const uint64_t x2 = mulhi(x, x), x3 = mulhi(x2, x);
                const uint64_t half = (uint64_t)(((u128)x2 + x3) >> 1);
                return (uint64_t)(((u128)half * 255) >> 8) + (x >> 8);
            }
            case 3: {
                const uint64_t sx = (uint64_t)(((u128)3 << 64) / 5), sy = (uint64_t)(((u128)3 << 64) / 10);
                return x < sx ? x >> 1 : sy + (uint64_t)(((u128)(x - sx) * 7) >> 2);
            }
            default: {
                const uint64_t i = x >> 48, f = x & ((uint64_t{1} << 48) - 1);
                return opt[i] + (uint64_t)(((u128)(opt[i + 1] - opt[i]) * f) >> 48);
            }
        }
    }
    // bucket within the part of hash h (whose part the caller knows)
    uint64_t bucket(uint64_t h) const { return mulhi(sh.B, gamma(sh.P * h)); }
    uint64_t part(uint64_t h) const { return mulhi(sh.P, h); }
    // slot within the part: reduce(y) (reduce.hpp:68-72) — the exact y mod S either way
    uint32_t slot(uint64_t y) const {
        if (p2) return (uint32_t)(mulhi(kMix, y) & (sh.S - 1));
        uint64_t r = y - mulhi(y, fm) * sh.S;
        while (r >= sh.S) r -= sh.S;
        return (uint32_t)r;
    }
};

// ---- the per-part hash-and-displace search (engine.hpp:105-292) -------------------------

struct PartResult {
    std::vector<uint64_t> free_slots;      // global slots < n left empty
    std::vector<uint64_t> overflow_slots;  // global slots >= n holding a key
};

struct Stats {
    uint64_t evictions = 0;
    uint64_t by_pct[100] = {};
};

class PartPlacer {
  public:
    PartPlacer(const Arith& a, uint64_t seed) : a_(a) {
        for (int p = 0; p < 256; p++) hp_[p] = kMix * ((uint64_t)p ^ seed);  // hash_pilot
        taken_.resize(a.sh.S / 64 + 1);
        owner_.resize(a.sh.S);
        start_.resize(a.sh.B + 1);
        first_.resize(a.sh.B);
    }

    // hashes: the part's sorted hashes. pilots: the part's B pilots. false = part failed
    // (the attempt reseeds), or `stop` was raised by another part.
    bool run(uint64_t part, const uint64_t* h, uint64_t m, uint8_t* pilots, PartResult& out,
             Stats& st, const std::atomic<bool>& stop) {
        const uint64_t S = a_.sh.S, B = a_.sh.B;
        std::fill(taken_.begin(), taken_.end(), 0);
        std::fill(owner_.begin(), owner_.end(), kNone);
        std::fill(first_.begin(), first_.end(), 0);
        std::memset(pilots, 0, B);
        h_ = h;
        // bucket boundaries: bucket ids are non-decreasing over sorted hashes
        uint64_t b = 0;
        start_[0] = 0;
        for (uint64_t i = 0; i < m; i++) {
            const uint64_t bi = a_.bucket(h[i]);
            while (b < bi) start_[++b] = (uint32_t)i;
        }
        while (b < B) start_[++b] = (uint32_t)m;
        // visiting order: size descending, id ascending (the heap order of engine.hpp:335)
        uint32_t maxsz = 0;
        for (uint64_t i = 0; i < B; i++) maxsz = std::max(maxsz, size(i));
        std::vector<uint32_t> bysz(maxsz + 2, 0);
        for (uint64_t i = 0; i < B; i++) bysz[size(i)]++;
        uint64_t nonempty = 0;
        {
            uint64_t at = 0;
            for (int64_t s = maxsz; s >= 1; s--) {
                const uint32_t c = bysz[s];
                bysz[s] = (uint32_t)at;
                at += c;
            }
            nonempty = at;
        }
        order_.resize(nonempty);
        for (uint64_t i = 0; i < B; i++)
            if (size(i)) order_[bysz[size(i)]++] = (uint32_t)i;
        std::priority_queue<uint64_t> evicted;  // keys (size << 32) | ~id
        uint64_t cursor = 0;
        uint32_t recent[kRecent];
        std::fill(recent, recent + kRecent, kNone);
        int rpos = 0;
        const uint64_t budget = 10 * S;
        uint64_t part_ev = 0, placed_first = 0, pops = 0;
        while (cursor < nonempty || !evicted.empty()) {
            if ((++pops & 1023) == 0 && stop.load(std::memory_order_relaxed)) return false;
            uint32_t bk;
            if (!evicted.empty() && (cursor == nonempty || evicted.top() > key(order_[cursor]))) {
                bk = UINT32_MAX - (uint32_t)evicted.top();
                evicted.pop();
            } else {
                bk = order_[cursor++];
            }
            const uint32_t k = size(bk);
            const uint64_t* kh = h + start_[bk];
            bool evict = false;
            int p = free_pilot(kh, k);
            if (p < 0) {
                p = cheapest_pilot(kh, k, recent);
                evict = true;
                if (p < 0) return false;  // every pilot self-collides or hits a recent bucket
            }
            pilots[bk] = (uint8_t)p;
            if (evict) {
                for (uint32_t i = 0; i < k; i++) {
                    const uint32_t s = slots_[i], v = owner_[s];
                    if (v != kNone) {  // displace v entirely
                        const uint64_t vhp = hp_[pilots[v]];
                        for (uint32_t j = start_[v]; j < start_[v + 1]; j++) {
                            const uint32_t vs = a_.slot(h[j] ^ vhp);
                            taken_[vs >> 6] &= ~(uint64_t{1} << (vs & 63));
                            owner_[vs] = kNone;
                        }
                        evicted.push(key(v));
                        part_ev++;
                        st.evictions++;
                        st.by_pct[std::min<uint64_t>(99, placed_first * 100 / std::max<uint64_t>(1, nonempty))]++;
                        if (part_ev > budget) return false;
                    }
                    taken_[s >> 6] |= uint64_t{1} << (s & 63);
                    owner_[s] = bk;
                }
                recent[rpos] = bk;
                rpos = (rpos + 1) % kRecent;
            } else {
                for (uint32_t i = 0; i < k; i++) {
                    taken_[slots_[i] >> 6] |= uint64_t{1} << (slots_[i] & 63);
                    owner_[slots_[i]] = bk;
                }
            }
            if (!first_[bk]) {
                first_[bk] = 1;
                placed_first++;
            }
        }
        // free slots below n and occupied slots at or above n, ascending (engine.hpp:324-343)
        const uint64_t base = part * S, n = a_.sh.n;
        out.free_slots.clear();
        out.overflow_slots.clear();
        for (uint64_t s = 0; s < S; s++) {
            const bool t = (taken_[s >> 6] >> (s & 63)) & 1;
            if (t && base + s >= n) out.overflow_slots.push_back(base + s);
            else if (!t && base + s < n) out.free_slots.push_back(base + s);
        }
        return true;
    }

  private:
    uint32_t size(uint64_t b) const { return start_[b + 1] - start_[b]; }
    static uint64_t key(uint32_t b, uint32_t sz) { return ((uint64_t)sz << 32) | (UINT32_MAX - b); }
    uint64_t key(uint32_t b) const { return key(b, size(b)); }
    bool is_taken(uint32_t s) const { return (taken_[s >> 6] >> (s & 63)) & 1; }

    bool distinct(const uint32_t* s, uint32_t k) const {
        for (uint32_t i = 1; i < k; i++)
            for (uint32_t j = 0; j < i; j++)
                if (s[i] == s[j]) return false;
        return true;
    }

    // smallest pilot whose slots are free and pairwise distinct (engine.hpp:131-147)
    int free_pilot(const uint64_t* kh, uint32_t k) {
        if (slots_.size() < k) slots_.resize(k), tmp_.resize(k);
        for (int p = 0; p < 256; p++) {
            const uint64_t hp = hp_[p];
            uint32_t i = 0;
            for (; i < k; i++) {
                const uint32_t s = a_.slot(kh[i] ^ hp);
                if (is_taken(s)) break;
                slots_[i] = s;
            }
            if (i == k && distinct(slots_.data(), k)) return p;
        }
        return -1;
    }

    // least total squared size of the buckets it would displace, never a recent displacer;
    // ties to the smaller pilot (engine.hpp:149-178). Leaves that pilot's slots in slots_.
    int cheapest_pilot(const uint64_t* kh, uint32_t k, const uint32_t* recent) {
        int best = -1;
        uint64_t best_cost = UINT64_MAX;
        for (int p = 0; p < 256; p++) {
            const uint64_t hp = hp_[p];
            for (uint32_t i = 0; i < k; i++) tmp_[i] = a_.slot(kh[i] ^ hp);
            if (!distinct(tmp_.data(), k)) continue;
            uint64_t cost = 0;
            bool ok = true;
            for (uint32_t i = 0; i < k && ok; i++) {
                const uint32_t o = owner_[tmp_[i]];
                if (o == kNone) continue;
                for (int r = 0; r < kRecent; r++)
                    if (recent[r] == o) {
                        ok = false;
                        break;
                    }
                if (!ok) break;
                const uint64_t sz = size(o);
                cost += sz * sz;
                if (cost >= best_cost) ok = false;  // cannot beat the incumbent
            }
            if (ok && cost < best_cost) {
                best_cost = cost;
                best = p;
                std::copy(tmp_.begin(), tmp_.begin() + k, slots_.begin());
            }
        }
        return best;
    }

    const Arith& a_;
    uint64_t hp_[256];
    const uint64_t* h_ = nullptr;
    std::vector<uint64_t> taken_;
    std::vector<uint32_t> owner_, start_, order_, slots_, tmp_;
    std::vector<uint8_t> first_;
};

// ---- remap table (remap.cpp:7-59, cacheline_ef.cpp:33-67, elias_fano.cpp:11-49) ---------

// F[q_i - n] = L_i for the i-th overflow slot q_i and free slot L_i; other positions repeat
// the previous defined value (L_0 before the first).
std::vector<uint64_t> remap_values(const std::vector<uint64_t>& fr, const std::vector<uint64_t>& ov,
                                   uint64_t n, uint64_t total) {
    if (fr.size() != ov.size()) throw BuildFail(PH_E_INVALID, "remap: |free| != |overflow|");
    std::vector<uint64_t> v(total - n, 0);
    if (fr.empty()) return v;
    uint64_t cur = fr[0];
    size_t j = 0;
    for (uint64_t i = 0; i < v.size(); i++) {
        if (j < ov.size() && ov[j] - n == i) cur = fr[j++];
        v[i] = cur;
    }
    return v;
}

void put32(std::vector<uint8_t>& o, uint32_t v) {
    const size_t at = o.size();
    o.resize(at + 4);
    std::memcpy(o.data() + at, &v, 4);
}
void put64(std::vector<uint8_t>& o, uint64_t v) {
    const size_t at = o.size();
    o.resize(at + 8);
    std::memcpy(o.data() + at, &v, 8);
}

// One 64-byte block: LE32 base = v_0 >> 8 at 0, 128-bit LE mask at 4 with bit
// i + (v_i >> 8) - base set, low bytes at 20. false if the values do not fit.
bool clef_block(const uint64_t* v, size_t c, uint8_t* out) {
    if (c == 0 || c > 44) return false;
    for (size_t i = 0; i < c; i++)
        if (v[i] >= (uint64_t{1} << 40)) return false;
    if (v[c - 1] - v[0] > (128 - 44) * 256) return false;
    const uint64_t base = v[0] >> 8;
    uint64_t mask[2] = {0, 0};
    for (size_t i = 0; i < c; i++) {
        const uint64_t bit = i + ((v[i] >> 8) - base);
        if (bit >= 128) return false;
        mask[bit >> 6] |= uint64_t{1} << (bit & 63);
    }
    std::memset(out, 0, 64);
    const uint32_t b32 = (uint32_t)base;
    std::memcpy(out, &b32, 4);
    std::memcpy(out + 4, mask, 16);
    for (size_t i = 0; i < c; i++) out[20 + i] = (uint8_t)(v[i] & 0xff);
    return true;
}

// Elias-Fano over values <= universe: low bits l = floor(log2(universe / count)) when that
// ratio exceeds 1; high part unary at (v >> l) + i; a sample (word << 16 | rank in word)
// every 512 values.
void elias_fano_payload(const std::vector<uint64_t>& v, uint64_t universe, std::vector<uint8_t>& o) {
    const uint64_t c = v.size();
    put64(o, c);
    put64(o, universe);
    if (c == 0) {
        o.push_back(0);
        put64(o, 0);
        put64(o, 0);
        put64(o, 0);
        return;
    }
    const uint64_t u = universe ? universe : 1;
    uint32_t l = 0;
    if (u / c > 1) l = 63 - __builtin_clzll(u / c);
    std::vector<uint64_t> low((c * l + 63) / 64 + 1, 0);
    std::vector<uint64_t> high(((u >> l) + c + 1 + 63) / 64 + 1, 0);
    std::vector<uint64_t> samples;
    for (uint64_t i = 0; i < c; i++) {
        if (l) {
            const uint64_t bp = i * l, lv = v[i] & ((uint64_t{1} << l) - 1);
            low[bp / 64] |= lv << (bp % 64);
            if (bp % 64 + l > 64) low[bp / 64 + 1] |= lv >> (64 - bp % 64);
        }
        const uint64_t hp = (v[i] >> l) + i;
        if (i % 512 == 0) samples.push_back(((hp / 64) << 16) | (uint64_t)__builtin_popcountll(high[hp / 64]));
        high[hp / 64] |= uint64_t{1} << (hp % 64);
    }
    o.push_back((uint8_t)l);
    for (const auto* a : {&low, &high, &samples}) {
        put64(o, a->size());
        for (uint64_t x : *a) put64(o, x);
    }
}

// Encodes the remap payload; returns the remap kind actually used (CacheLineEF falls back
// to plain32 when any block does not fit, remap.cpp:27-44).
int remap_payload(int kind, const std::vector<uint64_t>& v, uint64_t n, std::vector<uint8_t>& o,
                  bool* fell_back) {
    *fell_back = false;
    if (kind == 1) {
        const size_t blocks = (v.size() + 43) / 44;
        o.assign(blocks * 64, 0);
        bool ok = true;
        for (size_t b = 0; b < blocks && ok; b++)
            ok = clef_block(v.data() + b * 44, std::min<size_t>(44, v.size() - b * 44), o.data() + b * 64);
        if (ok) return 1;
        *fell_back = true;
        o.clear();
        kind = 0;
    }
    if (kind == 2) {
        for (size_t i = 0; i < v.size(); i++)
            if ((i && v[i] < v[i - 1]) || v[i] > n) throw BuildFail(PH_E_INVALID, "elias-fano: bad remap values");
        elias_fano_payload(v, n, o);
        return 2;
    }
    if (n > (uint64_t{1} << 32)) throw BuildFail(PH_E_INVALID, "plain remap array needs n <= 2^32");
    o.resize(v.size() * 4);
    for (size_t i = 0; i < v.size(); i++) {
        const uint32_t x = (uint32_t)v[i];
        std::memcpy(o.data() + 4 * i, &x, 4);
    }
    return 0;
}

// PTRH v1 (serde.hpp:12-31, serialize: serde.cpp:142-170)
std::vector<uint8_t> ptrh_bytes(const Shape& sh, const ph_build_params& p, uint64_t seed,
                                int remap_kind, const std::vector<uint8_t>& pilots,
                                const std::vector<uint8_t>& remap, uint8_t key_kind = 0,
                                uint8_t hash_algo = 0) {
    std::vector<uint8_t> o;
    o.reserve(72 + pilots.size() + remap.size());
    o.insert(o.end(), {'P', 'T', 'R', 'H'});
    put32(o, 1);
    o.insert(o.end(), {key_kind /*0 u64, 1 bytes*/, hash_algo /*0 fx64, 1 aes64, 3 portable64*/, p.bucket_fn,
                       (uint8_t)remap_kind, p.reduce_kind, 0, 0, 0});
    for (uint64_t x : {sh.n, sh.P, sh.S, sh.B, seed, (uint64_t)pilots.size(), (uint64_t)remap.size()})
        put64(o, x);
    o.insert(o.end(), pilots.begin(), pilots.end());
    o.insert(o.end(), remap.begin(), remap.end());
    return o;
}

double ms_since(std::chrono::steady_clock::time_point t) {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t).count();
}

unsigned thread_count(unsigned t) {
    if (t) return t;
    const unsigned hw = std::thread::hardware_concurrency();
    return hw ? hw : 1;
}

// Where the parts' sorted hashes come from: host memory, or the device through a ring of
// pinned buffers that a copier thread fills in part order.
struct PartFeed {
    virtual ~PartFeed() = default;
    // the part's hashes; valid until release(part). Blocks until they are on the host.
    virtual const uint64_t* get(uint64_t part) = 0;
    virtual void release(uint64_t part) = 0;
    virtual void abort() {}
};

struct HostFeed : PartFeed {
    const uint64_t* h;
    const uint64_t* off;
    HostFeed(const uint64_t* h_, const uint64_t* o) : h(h_), off(o) {}
    const uint64_t* get(uint64_t p) override { return h + off[p]; }
    void release(uint64_t) override {}
};

struct DeviceFeed : PartFeed {
    static constexpr int kSlots = 4;
    const uint64_t* d_h;
    std::vector<uint64_t> off;  // host copy of the part offsets
    uint64_t P = 0, slot_words = 0;
    uint64_t* slots[kSlots] = {};
    cudaStream_t s = nullptr;
    std::mutex mu;
    std::condition_variable cv;
    int refs[kSlots] = {};
    std::vector<int> part_slot;
    std::vector<uint64_t> part_at;
    uint64_t ready = 0;
    bool stopped = false;
    cudaError_t err = cudaSuccess;
    std::thread copier;

    cudaError_t start(const uint64_t* d_hashes, const uint64_t* d_off, uint64_t parts) {
        d_h = d_hashes;
        P = parts;
        off.resize(P + 1);
        cudaError_t e = cudaMemcpy(off.data(), d_off, (P + 1) * 8, cudaMemcpyDeviceToHost);
        uint64_t maxpart = 0;
        for (uint64_t p = 0; p < P; p++) maxpart = std::max(maxpart, off[p + 1] - off[p]);
        slot_words = std::max<uint64_t>(uint64_t{16} << 20, maxpart);  // 128 MB
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
        for (int i = 0; i < kSlots && e == cudaSuccess; i++)
            e = cudaHostAlloc(reinterpret_cast<void**>(&slots[i]), slot_words * 8, cudaHostAllocDefault);
        if (e != cudaSuccess) return e;
        part_slot.assign(P, -1);
        part_at.assign(P, 0);
        int dev = 0;
        cudaGetDevice(&dev);
        copier = std::thread([this, dev] { run(dev); });
        return cudaSuccess;
    }
    void run(int dev) {
        cudaSetDevice(dev);
        uint64_t p = 0;
        int slot = 0;
        while (p < P) {
            uint64_t q = p + 1;
            while (q < P && off[q + 1] - off[p] <= slot_words) q++;
            {
                std::unique_lock<std::mutex> lk(mu);
                cv.wait(lk, [&] { return refs[slot] == 0 || stopped; });
                if (stopped) break;
            }
            cudaError_t e = cudaMemcpyAsync(slots[slot], d_h + off[p], (off[q] - off[p]) * 8,
                                            cudaMemcpyDeviceToHost, s);
            if (e == cudaSuccess) e = cudaStreamSynchronize(s);
            std::lock_guard<std::mutex> lk(mu);
            if (e != cudaSuccess) {
                err = e;
                stopped = true;
                cv.notify_all();
                break;
            }
            for (uint64_t r = p; r < q; r++) {
                part_slot[r] = slot;
                part_at[r] = off[r] - off[p];
            }
            refs[slot] = (int)(q - p);
            ready = q;
            cv.notify_all();
            p = q;
            slot = (slot + 1) % kSlots;
        }
    }
    const uint64_t* get(uint64_t p) override {
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [&] { return ready > p || stopped; });
        if (ready <= p) return nullptr;
        return slots[part_slot[p]] + part_at[p];
    }
    void release(uint64_t p) override {
        std::lock_guard<std::mutex> lk(mu);
        if (--refs[part_slot[p]] == 0) cv.notify_all();
    }
    void abort() override {
        std::lock_guard<std::mutex> lk(mu);
        stopped = true;
        cv.notify_all();
    }
    ~DeviceFeed() override {
        abort();
        if (copier.joinable()) copier.join();
        for (auto* b : slots)
            if (b) cudaFreeHost(b);
        if (s) cudaStreamDestroy(s);
    }
};

// Places every part (threads in parallel over parts, engine.hpp:476-541) and assembles the
// index. Returns false if a part failed (the caller reseeds).
bool place_all(const Arith& a, uint64_t seed, const uint64_t* off, PartFeed& feed, unsigned threads,
               bool copy_parts, std::vector<uint8_t>& pilots, std::vector<PartResult>& parts,
               Stats& st) {
    const Shape& sh = a.sh;
    pilots.assign(sh.P * sh.B, 0);
    parts.assign(sh.P, PartResult{});
    std::atomic<uint64_t> next{0};
    std::atomic<bool> stop{false};
    const unsigned T = (unsigned)std::min<uint64_t>(thread_count(threads), std::max<uint64_t>(1, sh.P));
    std::vector<Stats> local(T);
    std::vector<std::thread> ws;
    for (unsigned w = 0; w < T; w++) {
        ws.emplace_back([&, w] {
            PartPlacer placer(a, seed);
            std::vector<uint64_t> mine;
            while (!stop.load(std::memory_order_relaxed)) {
                const uint64_t p = next.fetch_add(1);
                if (p >= sh.P) break;
                const uint64_t m = off[p + 1] - off[p];
                const uint64_t* h = feed.get(p);
                if (!h) {  // the feed stopped (transfer error or another part failed)
                    stop = true;
                    break;
                }
                if (copy_parts) {  // out of the pinned ring, so its slot can refill
                    mine.assign(h, h + m);
                    feed.release(p);
                    h = mine.data();
                }
                if (!placer.run(p, h, m, pilots.data() + p * sh.B, parts[p], local[w], stop)) {
                    stop = true;
                    feed.abort();  // wake workers waiting for later parts
                    break;
                }
            }
        });
    }
    for (auto& t : ws) t.join();
    if (stop.load()) {
        feed.abort();
        return false;
    }
    for (const Stats& l : local) {
        st.evictions += l.evictions;
        for (int i = 0; i < 100; i++) st.by_pct[i] += l.by_pct[i];
    }
    return true;
}

// The remap table's payload from the parts' free / overflow slot lists (engine.hpp:544-557).
int remap_stage(const Shape& sh, const ph_build_params& p, const std::vector<PartResult>& parts,
                std::vector<uint8_t>& payload, ph_build_stats* stats) {
    std::vector<uint64_t> fr, ov;
    for (const auto& r : parts) {
        fr.insert(fr.end(), r.free_slots.begin(), r.free_slots.end());
        ov.insert(ov.end(), r.overflow_slots.begin(), r.overflow_slots.end());
    }
    const std::vector<uint64_t> v = remap_values(fr, ov, sh.n, sh.P * sh.S);
    bool fell_back = false;
    const int kind = remap_payload(p.remap_kind, v, sh.n, payload, &fell_back);
    if (stats) {
        stats->remap_kind = (uint8_t)kind;
        stats->remap_fell_back = fell_back;
        stats->pilot_bytes = sh.P * sh.B;
        stats->remap_payload_bytes = payload.size();
    }
    return kind;
}

std::vector<uint8_t> finish(const Shape& sh, const ph_build_params& p, uint64_t seed,
                            const std::vector<uint8_t>& pilots, const std::vector<PartResult>& parts,
                            ph_build_stats* stats, uint8_t key_kind = 0, uint8_t hash_algo = 0) {
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<uint8_t> payload;
    const int kind = remap_stage(sh, p, parts, payload, stats);
    std::vector<uint8_t> out = ptrh_bytes(sh, p, seed, kind, pilots, payload, key_kind, hash_algo);
    if (stats) stats->remap_ms = ms_since(t0);
    return out;
}

Arith make_arith(const Shape& sh, const ph_build_params& p, const std::vector<uint64_t>& opt) {
    Arith a{sh, p.bucket_fn, opt.empty() ? nullptr : opt.data(), pow2(sh.S), 0};
    if (!a.p2) a.fm = UINT64_MAX / sh.S;
    return a;
}

// Where the pilot search of ph_gpu_build_u64 runs: 0 = on the GPU when the shape allows it
// (ph_search.cu), else on host threads; 1 = always host threads; 2 = GPU or PH_E_UNSUPPORTED.
std::atomic<int> g_search_mode{0};

// The free / overflow slot lists of every part from the GPU search's occupancy bitmaps
// (engine.hpp:324-343), parts in parallel.
void results_from_bitmaps(const Shape& sh, const std::vector<uint32_t>& taken, uint32_t words,
                          unsigned threads, std::vector<PartResult>& parts) {
    parts.assign(sh.P, PartResult{});
    std::atomic<uint64_t> next{0};
    const unsigned T = (unsigned)std::min<uint64_t>(thread_count(threads), std::max<uint64_t>(1, sh.P));
    std::vector<std::thread> ws;
    for (unsigned t = 0; t < T; t++)
        ws.emplace_back([&] {
            for (;;) {
                const uint64_t p = next.fetch_add(1);
                if (p >= sh.P) break;
                const uint32_t* tk = taken.data() + p * words;
                const uint64_t base = p * sh.S;
                PartResult& out = parts[p];
                for (uint64_t s0 = 0; s0 < sh.S; s0 += 32) {
                    const uint32_t wv = tk[s0 >> 5];
                    const uint32_t lim = (uint32_t)std::min<uint64_t>(32, sh.S - s0);
                    if (base + s0 + lim <= sh.n) {  // all below n: the free ones
                        uint32_t fr = ~wv & (lim == 32 ? 0xffffffffu : (1u << lim) - 1);
                        while (fr) {
                            out.free_slots.push_back(base + s0 + (uint32_t)__builtin_ctz(fr));
                            fr &= fr - 1;
                        }
                    } else {
                        for (uint32_t b = 0; b < lim; b++) {
                            const bool t1 = (wv >> b) & 1;
                            const uint64_t g = base + s0 + b;
                            if (t1 && g >= sh.n) out.overflow_slots.push_back(g);
                            else if (!t1 && g < sh.n) out.free_slots.push_back(g);
                        }
                    }
                }
            }
        });
    for (auto& t : ws) t.join();
}

// Host keys -> device. A plain cudaMemcpy from pageable memory runs at ~11 GB/s (0.7 s for
// the 8 GB of config 3); here host threads copy 16 MiB pieces into their own pinned buffers
// and send them with async copies, two buffers per thread, so the transfer runs at the PCIe
// rate (the host memcpy of one piece overlaps the DMA of the previous ones).
cudaError_t upload_pipelined(uint64_t* d, const uint64_t* h, size_t n, unsigned threads, int device) {
    constexpr size_t kPiece = size_t{2} << 20;  // words: 16 MiB
    if (n < 4 * kPiece) return cudaMemcpy(d, h, n * 8, cudaMemcpyHostToDevice);
    const size_t pieces = (n + kPiece - 1) / kPiece;
    const unsigned T = (unsigned)std::min<size_t>(std::min(8u, thread_count(threads)), pieces);
    std::atomic<size_t> next{0};
    std::atomic<int> err{(int)cudaSuccess};
    uint64_t* pin_all = nullptr;  // one page-locked region, two pieces per thread
    cudaError_t ea = cudaHostAlloc(reinterpret_cast<void**>(&pin_all), (size_t)T * 2 * kPiece * 8, cudaHostAllocDefault);
    if (ea != cudaSuccess) {
        cudaGetLastError();
        return cudaMemcpy(d, h, n * 8, cudaMemcpyHostToDevice);
    }
    std::vector<std::thread> ws;
    for (unsigned t = 0; t < T; t++)
        ws.emplace_back([&, t] {
            auto fail = [&](cudaError_t e) {
                int ok = (int)cudaSuccess;
                if (e != cudaSuccess) err.compare_exchange_strong(ok, (int)e);
                return e != cudaSuccess;
            };
            if (fail(cudaSetDevice(device))) return;
            uint64_t* pin[2] = {pin_all + (size_t)t * 2 * kPiece, pin_all + ((size_t)t * 2 + 1) * kPiece};
            cudaStream_t st = nullptr;
            cudaEvent_t ev[2] = {nullptr, nullptr};
            bool ok = !fail(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
            for (int b = 0; b < 2 && ok; b++) ok = !fail(cudaEventCreateWithFlags(&ev[b], cudaEventDisableTiming));
            for (size_t k = 0; ok && err.load() == (int)cudaSuccess; k++) {
                const size_t i = next.fetch_add(1);
                if (i >= pieces) break;
                const int b = (int)(k & 1);
                const size_t w0 = i * kPiece, len = std::min(kPiece, n - w0);
                if (k >= 2 && fail(cudaEventSynchronize(ev[b]))) break;
                std::memcpy(pin[b], h + w0, len * 8);
                if (fail(cudaMemcpyAsync(d + w0, pin[b], len * 8, cudaMemcpyHostToDevice, st))) break;
                if (fail(cudaEventRecord(ev[b], st))) break;
            }
            if (st) fail(cudaStreamSynchronize(st));
            for (int b = 0; b < 2; b++)
                if (ev[b]) cudaEventDestroy(ev[b]);
            if (st) cudaStreamDestroy(st);
        });
    for (auto& t : ws) t.join();
    cudaFreeHost(pin_all);
    return (cudaError_t)err.load();
}

Shape resolve_shape(uint64_t n, const ph_build_params& p) {
    if (!p.parts && !p.slots_per_part && !p.buckets_per_part) return make_shape(n, p);
    // build_with_shape (construction.cpp:145-152)
    if (!p.parts || !p.slots_per_part || !p.buckets_per_part)
        throw BuildFail(PH_E_INVALID, "a forced shape needs parts, slots_per_part and buckets_per_part");
    if ((u128)p.parts * p.slots_per_part < n) throw BuildFail(PH_E_INVALID, "shape has fewer slots than keys");
    if (!pow2(p.slots_per_part) && p.slots_per_part >= (uint64_t{1} << 32))
        throw BuildFail(PH_E_INVALID, "reduce: fastmod needs S < 2^32");
    return Shape{n, p.parts, p.slots_per_part, p.buckets_per_part};
}

uint8_t* to_malloc(const std::vector<uint8_t>& v) {
    uint8_t* o = static_cast<uint8_t*>(std::malloc(std::max<size_t>(1, v.size())));
    if (o) std::memcpy(o, v.data(), v.size());
    return o;
}

bool is_device_ptr(const void* p) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

template <class F>
int guarded(F&& f) {
    try {
        return f();
    } catch (const BuildFail& e) {
        return phg::report_error(e.code, e.what());
    } catch (const std::bad_alloc&) {
        return phg::report_error(PH_E_NOMEM, "host allocation failed");
    } catch (const std::exception& e) {
        return phg::report_error(PH_E_INVALID, e.what());
    }
}

}  // namespace

extern "C" {

int ph_build_preset(const char* name, ph_build_params* out) {
    if (!name || !out) return phg::report_error(PH_E_INVALID, "null argument");
    // preset() (shape.cpp:65-84)
    ph_build_params p{};
    p.alpha_num = 99;
    p.alpha_den = 100;
    p.reduce_kind = 2;
    p.max_seed_retries = 10;
    p.seed = kGolden;
    if (!std::strcmp(name, "fast")) {
        p.bucket_fn = 0, p.lambda_num = 30, p.lambda_den = 10, p.remap_kind = 0;
    } else if (!std::strcmp(name, "default")) {
        p.bucket_fn = 2, p.lambda_num = 35, p.lambda_den = 10, p.remap_kind = 1;
    } else if (!std::strcmp(name, "compact")) {
        p.bucket_fn = 2, p.lambda_num = 40, p.lambda_den = 10, p.remap_kind = 1;
    } else {
        return phg::report_error(PH_E_INVALID, std::string("unknown preset: ") + name);
    }
    *out = p;
    return PH_OK;
}

int ph_build_compute_shape(uint64_t n, const ph_build_params* params, uint64_t* parts,
                           uint64_t* slots_per_part, uint64_t* buckets_per_part) {
    if (!params || !parts || !slots_per_part || !buckets_per_part)
        return phg::report_error(PH_E_INVALID, "null argument");
    return guarded([&] {
        validate(*params);
        if (!n) throw BuildFail(PH_E_INVALID, "n must be >= 1");
        const Shape s = make_shape(n, *params);
        *parts = s.P, *slots_per_part = s.S, *buckets_per_part = s.B;
        return PH_OK;
    });
}

int ph_build_from_sorted_u64(const uint64_t* hashes, const uint64_t* offsets, size_t n,
                             const ph_build_params* params, uint64_t seed, unsigned threads,
                             uint8_t** ptrh, size_t* len, ph_build_stats* stats) {
    PH_RANGE("ph_build_from_sorted_u64");
    if ((!hashes && n) || !offsets || !params || !ptrh || !len)
        return phg::report_error(PH_E_INVALID, "null argument");
    return guarded([&] {
        validate(*params);
        if (!n) throw BuildFail(PH_E_INVALID, "key set is empty");
        const Shape sh = resolve_shape(n, *params);
        if (offsets[sh.P] != n) throw BuildFail(PH_E_INVALID, "offsets[parts] != n");
        for (uint64_t p = 0; p < sh.P; p++)
            if (offsets[p + 1] < offsets[p] || offsets[p + 1] - offsets[p] > sh.S)
                throw BuildFail(PH_E_BUILD_FAILED, "a part holds more keys than slots");
        std::vector<uint64_t> opt;
        if (params->bucket_fn == 4) phg::optimal_gamma_table(opt);
        const Arith a = make_arith(sh, *params, opt);
        const auto t0 = std::chrono::steady_clock::now();
        HostFeed feed(hashes, offsets);
        std::vector<uint8_t> pilots;
        std::vector<PartResult> parts;
        Stats st;
        if (!place_all(a, seed, offsets, feed, threads, false, pilots, parts, st))
            throw BuildFail(PH_E_BUILD_FAILED, "a part failed under this seed");
        if (stats) {
            *stats = ph_build_stats{};
            stats->search_ms = ms_since(t0);
        }
        const std::vector<uint8_t> out = finish(sh, *params, seed, pilots, parts, stats);
        if (stats) {
            stats->n = n, stats->parts = sh.P, stats->slots_per_part = sh.S, stats->buckets_per_part = sh.B;
            stats->seed = seed, stats->attempts = 1, stats->total_evictions = st.evictions;
            std::memcpy(stats->evictions_by_percentile, st.by_pct, sizeof(st.by_pct));
            stats->total_ms = ms_since(t0);
        }
        if (!(*ptrh = to_malloc(out))) throw std::bad_alloc();
        *len = out.size();
        return PH_OK;
    });
}

}  // extern "C"

namespace {
// What differs between key kinds in a build: where the attempt's u64 keys come from (u64
// keys: the input itself; byte strings: per seed, the pre-images key' with
// C * (key' ^ seed) == hash_bytes(key, seed).lo, so that the u64 front reproduces the string
// hashes), the header's key kind and hash id, and what equal hashes mean.
struct KeyFeed {
    uint8_t key_kind = 0, hash_algo = 0;
    bool dup_is_error = true;  // u64: equal hashes are equal keys (construction.cpp:128-133)
    // host -> device staging before the attempts; returns the time it took in upload_ms
    std::function<void(unsigned threads, int device)> upload;
    std::function<const uint64_t*(uint64_t seed, int sms)> keys_for_seed;
};

int build_impl(size_t n, const ph_build_params* params, unsigned threads, int device, KeyFeed& src,
               uint8_t** ptrh, size_t* len, ph_build_stats* stats) {
    int prev = -1;
    cudaGetDevice(&prev);
    if (prev != device && cudaSetDevice(device) != cudaSuccess)
        return phg::report_error(PH_E_CUDA, "cudaSetDevice failed");
    struct Restore {
        int prev, dev;
        ~Restore() {
            if (prev >= 0 && prev != dev) cudaSetDevice(prev);
        }
    } restore{prev, device};
    uint64_t* d_h = nullptr;
    uint64_t* d_off = nullptr;
    const int rc = guarded([&] {
        validate(*params);
        if (!n) throw BuildFail(PH_E_INVALID, "key set is empty");
        const Shape sh = resolve_shape(n, *params);
        std::vector<uint64_t> opt;
        if (params->bucket_fn == 4) phg::optimal_gamma_table(opt);
        const auto t0 = std::chrono::steady_clock::now();
        auto cuda = [](cudaError_t e, const char* what) {
            if (e == cudaErrorMemoryAllocation) throw BuildFail(PH_E_NOMEM, what);
            if (e != cudaSuccess) throw BuildFail(PH_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
        };
        src.upload(threads, device);
        uint32_t duplicate_failures = 0;
        cuda(cudaMalloc(&d_h, n * 8), "device hash buffer");
        cuda(cudaMalloc(&d_off, (sh.P + 1) * 8), "device offsets");
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
        if (stats) *stats = ph_build_stats{};
        const double upload_ms = ms_since(t0);
        double prep_ms = 0, search_ms = 0;
        uint64_t seed = params->seed;
        for (uint32_t attempt = 0; attempt <= params->max_seed_retries; attempt++) {
            // build_u64_impl's attempt loop (construction.cpp:113-138)
            PH_RANGE("build attempt");
            auto tp = std::chrono::steady_clock::now();
            int status = 0;
            const uint64_t* dk = src.keys_for_seed(seed, sms);
            cuda(phg::build_prepare_u64(dk, n, sh.P, sh.S, seed, d_h, d_off, &status, nullptr, sms),
                 "build_prepare_u64");
            prep_ms += ms_since(tp);
            if (status == 2) {
                if (src.dup_is_error) throw BuildFail(PH_E_DUPLICATE, "duplicate keys in input");
                // byte strings (construction.cpp:208-216): equal keys or a fingerprint collision;
                // the reference reseeds and, the second time, widens to the 128-bit hash
                if (++duplicate_failures >= 2)
                    throw BuildFail(PH_E_UNSUPPORTED,
                                    "persistent duplicate 64-bit fingerprints (duplicate keys in input?): the "
                                    "reference widens to its 128-bit hash here, which this builder does not produce");
            }
            bool searched = false;
            if (status == 0 && g_search_mode.load() != 1) {
                // the pilot search on the GPU (ph_search.cu): one CTA per part
                std::vector<uint64_t> hoff(sh.P + 1);
                cuda(cudaMemcpy(hoff.data(), d_off, (sh.P + 1) * 8, cudaMemcpyDeviceToHost), "part offsets");
                uint64_t maxpart = 0;
                for (uint64_t p = 0; p < sh.P; p++) maxpart = std::max(maxpart, hoff[p + 1] - hoff[p]);
                const bool can = phg::search_parts_supported(sh.S, sh.B, maxpart);
                if (!can && g_search_mode.load() == 2)
                    throw BuildFail(PH_E_UNSUPPORTED, "the GPU pilot search does not take this shape");
                if (can) {
                    tp = std::chrono::steady_clock::now();
                    const uint32_t words = (uint32_t)((sh.S + 31) / 32);
                    uint8_t* d_pilots = nullptr;
                    uint32_t* d_taken = nullptr;
                    uint64_t* d_opt = nullptr;
                    struct Free {
                        uint8_t*& a;
                        uint32_t*& b;
                        uint64_t*& c;
                        ~Free() {
                            if (a) cudaFree(a);
                            if (b) cudaFree(b);
                            if (c) cudaFree(c);
                        }
                    } fr{d_pilots, d_taken, d_opt};
                    cuda(cudaMalloc(&d_pilots, sh.P * sh.B), "device pilots");
                    cuda(cudaMalloc(&d_taken, sh.P * (uint64_t)words * 4), "device occupancy bitmaps");
                    if (!opt.empty()) {
                        cuda(cudaMalloc(&d_opt, opt.size() * 8), "device gamma table");
                        cuda(cudaMemcpy(d_opt, opt.data(), opt.size() * 8, cudaMemcpyHostToDevice), "gamma table");
                    }
                    unsigned long long hst[4] = {}, hpct[100] = {};
                    const bool trace = std::getenv("PH_GPU_BUILD_TRACE") != nullptr;
                    const double t_alloc = ms_since(tp);
                    cuda(phg::search_parts_gpu(d_h, d_off, n, sh.P, sh.S, sh.B, seed, params->bucket_fn, d_opt,
                                               maxpart, d_pilots, d_taken, hst, hpct, nullptr, sms),
                         "search_parts_gpu");
                    const double t_kernel = ms_since(tp);
                    if (hst[1] && g_search_mode.load() == 2)
                        throw BuildFail(PH_E_UNSUPPORTED, "the GPU pilot search gave up on this key set");
                    if (!hst[1]) {
                        searched = true;
                        if (!hst[0]) {  // every part placed
                            std::vector<uint32_t> taken(sh.P * (uint64_t)words);
                            cuda(cudaMemcpy(taken.data(), d_taken, taken.size() * 4, cudaMemcpyDeviceToHost),
                                 "occupancy bitmaps");
                            const double t_copy = ms_since(tp);
                            std::vector<PartResult> parts;
                            results_from_bitmaps(sh, taken, words, threads, parts);
                            if (trace)
                                std::fprintf(stderr, "[ph_gpu build] search: alloc %.1f ms, kernel+workspace %.1f ms, "
                                             "bitmaps back %.1f ms, slot lists %.1f ms\n", t_alloc, t_kernel - t_alloc,
                                             t_copy - t_kernel, ms_since(tp) - t_copy);
                            search_ms += ms_since(tp);
                            // the remap table, then the PTRH bytes assembled in the returned
                            // buffer itself: the pilots come straight from the device
                            const auto tr = std::chrono::steady_clock::now();
                            std::vector<uint8_t> payload;
                            const int kind = remap_stage(sh, *params, parts, payload, stats);
                            const std::vector<uint8_t> head =
                                ptrh_bytes(sh, *params, seed, kind, {}, {}, src.key_kind, src.hash_algo);
                            const uint64_t pb = sh.P * sh.B;
                            std::vector<uint8_t> hdr(head);  // sizes of the empty sections -> real ones
                            std::memcpy(hdr.data() + 56, &pb, 8);
                            const uint64_t rl = payload.size();
                            std::memcpy(hdr.data() + 64, &rl, 8);
                            uint8_t* buf = static_cast<uint8_t*>(std::malloc(hdr.size() + pb + rl));
                            if (!buf) throw std::bad_alloc();
                            std::memcpy(buf, hdr.data(), hdr.size());
                            const cudaError_t ce = cudaMemcpy(buf + hdr.size(), d_pilots, pb, cudaMemcpyDeviceToHost);
                            if (ce != cudaSuccess) {
                                std::free(buf);
                                cuda(ce, "pilots");
                            }
                            std::memcpy(buf + hdr.size() + pb, payload.data(), rl);
                            if (stats) stats->remap_ms = ms_since(tr);
                            if (stats) {
                                stats->n = n, stats->parts = sh.P, stats->slots_per_part = sh.S;
                                stats->buckets_per_part = sh.B, stats->seed = seed, stats->attempts = attempt + 1;
                                stats->total_evictions = hst[3];
                                for (int i = 0; i < 100; i++) stats->evictions_by_percentile[i] = hpct[i];
                                stats->upload_ms = upload_ms, stats->prepare_ms = prep_ms;
                                stats->search_ms = search_ms, stats->total_ms = ms_since(t0);
                                stats->reserved[0] = 1;  // the search ran on the GPU
                            }
                            *ptrh = buf;
                            *len = hdr.size() + pb + rl;
                            return PH_OK;
                        }
                        search_ms += ms_since(tp);  // a part failed: reseed
                    }
                }
            }
            if (status == 0 && !searched) {
                tp = std::chrono::steady_clock::now();
                DeviceFeed feed;
                cuda(feed.start(d_h, d_off, sh.P), "hash transfer ring");
                const Arith a = make_arith(sh, *params, opt);
                std::vector<uint8_t> pilots;
                std::vector<PartResult> parts;
                Stats st;
                const bool ok = place_all(a, seed, feed.off.data(), feed, threads, true, pilots, parts, st);
                search_ms += ms_since(tp);
                if (feed.err != cudaSuccess) cuda(feed.err, "hash transfer");
                if (ok) {
                    const std::vector<uint8_t> out =
                        finish(sh, *params, seed, pilots, parts, stats, src.key_kind, src.hash_algo);
                    if (stats) {
                        stats->n = n, stats->parts = sh.P, stats->slots_per_part = sh.S;
                        stats->buckets_per_part = sh.B, stats->seed = seed, stats->attempts = attempt + 1;
                        stats->total_evictions = st.evictions;
                        std::memcpy(stats->evictions_by_percentile, st.by_pct, sizeof(st.by_pct));
                        stats->upload_ms = upload_ms, stats->prepare_ms = prep_ms;
                        stats->search_ms = search_ms, stats->total_ms = ms_since(t0);
                    }
                    if (!(*ptrh = to_malloc(out))) throw std::bad_alloc();
                    *len = out.size();
                    return PH_OK;
                }
            }
            seed = kMix * ((seed ^ attempt) ^ kGolden);  // next_seed (build.hpp:67-69)
        }
        throw BuildFail(PH_E_BUILD_FAILED, "construction failed after " +
                                               std::to_string(params->max_seed_retries + 1) +
                                               " seed attempts");
    });
    if (d_h) cudaFree(d_h);
    if (d_off) cudaFree(d_off);
    return rc;
}
}  // namespace

extern "C" {

int ph_gpu_build_u64(const uint64_t* keys, size_t n, const ph_build_params* params,
                     unsigned threads, int device, uint8_t** ptrh, size_t* len,
                     ph_build_stats* stats) {
    PH_RANGE("ph_gpu_build_u64");
    if ((!keys && n) || !params || !ptrh || !len) return phg::report_error(PH_E_INVALID, "null argument");
    uint64_t* d_keys = nullptr;
    KeyFeed feed;
    feed.upload = [&](unsigned th, int dev) {
        if (is_device_ptr(keys) || !n) return;
        const auto t0 = std::chrono::steady_clock::now();
        cudaError_t e = cudaMalloc(&d_keys, n * 8);
        if (e == cudaErrorMemoryAllocation) throw BuildFail(PH_E_NOMEM, "device key buffer");
        const double t_m = ms_since(t0);
        if (e == cudaSuccess) e = upload_pipelined(d_keys, keys, n, th, dev);
        if (e != cudaSuccess) throw BuildFail(PH_E_CUDA, std::string("key upload: ") + cudaGetErrorString(e));
        if (std::getenv("PH_GPU_BUILD_TRACE"))
            std::fprintf(stderr, "[ph_gpu build] key buffer cudaMalloc %.1f ms, upload %.1f ms\n", t_m,
                         ms_since(t0) - t_m);
    };
    feed.keys_for_seed = [&](uint64_t, int) { return d_keys ? d_keys : keys; };
    const int rc = build_impl(n, params, threads, device, feed, ptrh, len, stats);
    if (d_keys) cudaFree(d_keys);
    return rc;
}

int ph_gpu_build_bytes(const uint8_t* bytes, const uint64_t* offsets, size_t n,
                       const ph_build_params* params, int hash_algo, unsigned threads, int device,
                       uint8_t** ptrh, size_t* len, ph_build_stats* stats) {
    PH_RANGE("ph_gpu_build_bytes");
    if (!offsets || !params || !ptrh || !len) return phg::report_error(PH_E_INVALID, "null argument");
    if (hash_algo != 1 && hash_algo != 3)
        return phg::report_error(PH_E_UNSUPPORTED, "string builds use the 64-bit hashes: aes64 (1) or portable64 (3)");
    if (n >= (uint64_t{1} << 32))
        return phg::report_error(PH_E_UNSUPPORTED, "2^32 or more string keys need the 128-bit hash");
    uint8_t* d_bytes = nullptr;
    uint64_t* d_offs = nullptr;
    uint64_t* d_pk = nullptr;
    const uint8_t* db = bytes;
    const uint64_t* dof = offsets;
    // the inverse of the integer hash's multiplier mod 2^64 (Newton iteration; C is odd)
    uint64_t cinv = kMix;
    for (int i = 0; i < 6; i++) cinv *= 2 - kMix * cinv;
    KeyFeed feed;
    feed.key_kind = 1;
    feed.hash_algo = (uint8_t)hash_algo;
    feed.dup_is_error = false;
    feed.upload = [&](unsigned th, int dev) {
        auto cuda = [](cudaError_t e, const char* what) {
            if (e == cudaErrorMemoryAllocation) throw BuildFail(PH_E_NOMEM, what);
            if (e != cudaSuccess) throw BuildFail(PH_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
        };
        if (!is_device_ptr(offsets)) {
            for (size_t i = 0; i < n; i++)
                if (offsets[i + 1] < offsets[i]) throw BuildFail(PH_E_INVALID, "offsets must be non-decreasing");
            const uint64_t total = offsets[n] - offsets[0];
            if (total && !bytes) throw BuildFail(PH_E_INVALID, "null bytes");
            if (is_device_ptr(bytes)) throw BuildFail(PH_E_INVALID, "bytes and offsets must both be host or both device");
            cuda(cudaMalloc(&d_offs, (n + 1) * 8), "device offsets of the keys");
            cuda(upload_pipelined(d_offs, offsets, n + 1, th, dev), "offset upload");
            cuda(cudaMalloc(&d_bytes, total + 32), "device key bytes");
            // offsets index `bytes`; the device copy starts at offsets[0]
            const uint8_t* hb = bytes + offsets[0];
            if ((reinterpret_cast<uintptr_t>(hb) & 7) == 0 && total >= 8) {
                cuda(upload_pipelined(reinterpret_cast<uint64_t*>(d_bytes), reinterpret_cast<const uint64_t*>(hb),
                                      total / 8, th, dev),
                     "key byte upload");
                if (total & 7)
                    cuda(cudaMemcpy(d_bytes + (total & ~uint64_t{7}), hb + (total & ~uint64_t{7}), total & 7,
                                    cudaMemcpyHostToDevice),
                         "key byte upload");
            } else {
                cuda(cudaMemcpy(d_bytes, hb, total, cudaMemcpyHostToDevice), "key byte upload");
            }
            db = d_bytes - offsets[0];
            dof = d_offs;
        } else if (!is_device_ptr(bytes)) {
            throw BuildFail(PH_E_INVALID, "bytes and offsets must both be host or both device");
        }
        cuda(cudaMalloc(&d_pk, n * 8), "device hash pre-images");
    };
    feed.keys_for_seed = [&](uint64_t seed, int sms) -> const uint64_t* {
        phg::DevIndex ix{};
        ix.seed = seed;
        ix.hash_algo = hash_algo;
        {  // AES round keys of hash.cpp:116-119
            auto mix64 = [](uint64_t z) {
                z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
                z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
                return z ^ (z >> 31);
            };
            const uint64_t w0[2] = {seed + kGolden, seed ^ 0x8bb84b93962eacc9ULL};
            const uint64_t w1[2] = {(~seed) * 0x6c62272e07bb0143ULL, mix64(seed) ^ 0x2d358dccaa6c78a5ULL};
            for (int i = 0; i < 4; i++) {
                ix.aes_k0[i] = (uint32_t)(w0[i / 2] >> (32 * (i % 2)));
                ix.aes_k1[i] = (uint32_t)(w1[i / 2] >> (32 * (i % 2)));
            }
        }
        const cudaError_t e = phg::launch_hash_bytes(ix, db, dof, d_pk, n, cinv, nullptr, sms);
        if (e != cudaSuccess) throw BuildFail(PH_E_CUDA, std::string("string hash kernel: ") + cudaGetErrorString(e));
        return d_pk;
    };
    const int rc = build_impl(n, params, threads, device, feed, ptrh, len, stats);
    if (d_bytes) cudaFree(d_bytes);
    if (d_offs) cudaFree(d_offs);
    if (d_pk) cudaFree(d_pk);
    return rc;
}

int ph_gpu_set_build_search(int mode) {
    if (mode < 0 || mode > 2) return phg::report_error(PH_E_INVALID, "mode must be 0, 1 or 2");
    g_search_mode.store(mode);
    return PH_OK;
}

void ph_free(void* p) { std::free(p); }

}  // extern "C"
