// ph_search.cu — the per-part hash-and-displace pilot search on the GPU (construction,
// SURVEY §8f-3; off the query path).
//
// The reference searches one part at a time on a CPU thread (engine.hpp:105-292): buckets
// are visited by size (descending, then id ascending, evicted buckets re-entering through a
// priority queue), each takes the smallest pilot whose slots are all free and pairwise
// distinct, or, when none of the 256 pilots is free, the pilot that displaces the least
// total squared bucket size (never a recently displacing bucket) and evicts what it hits.
// The order of visits and every choice decide the pilots, so the search of a part is
// sequential; here ONE CTA SEARCHES ONE PART and the 256 pilots of the bucket being placed
// are tested at once, one per thread:
//
//   prologue   bucket boundaries of the part's sorted hashes (exact gamma), the visiting
//              order by a stable counting sort on bucket size, and the part's hashes copied
//              into visiting order, so the main loop streams them;
//   step       eight buckets at once, one per warp: lane p of a round hashes the bucket's keys
//              with pilot 32*round + p and tests the part's occupancy bitmap, which lives in
//              shared memory (S bits); the first round with a free pilot ends the warp's
//              search; the eight winners commit in visiting order (a claim per slot, rolled
//              back and redone serially if two buckets of the batch want one slot). Two CTA
//              barriers per eight buckets, no global-memory round trip on the common path;
//   full step  (an evicted bucket pending, or no pilot free) all 256 pilots of one bucket,
//              one per thread;
//   eviction   (0.6 % of buckets at lambda = 3) every thread prices its pilot from the
//              global owner[] array, a block argmin picks the cheapest, thread 0 displaces
//              the hit buckets exactly in the reference's order and pushes them on a small
//              shared-memory heap.
//
// The result (pilots and occupancy bitmaps) is what the host search in ph_builder.cu
// produces, bit for bit; tests/test_builder.py compares the built PTRH bytes with the
// reference's. Shapes this kernel does not take (S beyond the shared-memory bitmap, a bucket
// needing an eviction to place more than kMaxK keys, more than kHeapCap evicted buckets pending) are reported as unsupported
// and the caller runs the host search instead.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "ph_device.cuh"
#include "ph_kernels.h"

namespace phg {
namespace {

constexpr int kSThreads = 256;          // one thread per pilot value
constexpr uint32_t kMaxK = 32;          // buckets up to this size: one pilot per thread;
                                        // larger ones: the CTA tests one pilot at a time
constexpr uint32_t kHeapCap = 512;      // pending evicted buckets (shared-memory heap)
constexpr uint32_t kNoBucket = 0xffffffffu;  // engine.hpp:91
constexpr int kRecent = 16;             // engine.hpp:92

// Checked builds (-DPH_CHECKS, tools/checked_run.py): slots, visiting indices, bucket ids,
// hash positions and heap sizes are bounds-checked on the device; violations are counted and
// read back with ph_gpu_check_errors (compute-sanitizer cannot attach on this GPU pool).
#ifdef PH_CHECKS
__device__ unsigned long long g_schk[2];  // [0] violations, [1] source line of the first
#define PH_SCHECK(c)                                                                   \
    do {                                                                               \
        if (!(c) && atomicAdd(&g_schk[0], 1ull) == 0) g_schk[1] = __LINE__;           \
    } while (0)
#else
#define PH_SCHECK(c) \
    do {             \
    } while (0)
#endif

struct Arith {
    uint64_t P, S, B, seed, fm;  // fm = floor((2^64 - 1) / S)
    uint64_t hre_cap;            // entries of a workspace's hre[] (checked builds)
    const uint64_t* opt;
    int fn, p2;
    ModFast mf;                  // 32-bit form of y mod S for 2^13 <= S < 2^21 (ph_arith.cuh)
};

__device__ __forceinline__ uint64_t gamma_rt(const Arith& a, uint64_t x) {
    switch (a.fn) {
        case 0: return gamma<0>(x, a.opt);
        case 1: return gamma<1>(x, a.opt);
        case 2: return gamma<2>(x, a.opt);
        case 3: return gamma<3>(x, a.opt);
        default: return gamma<4>(x, a.opt);
    }
}
// bucket of hash h within its part: hi64(B * gamma(P * h)) (bucket_fn.hpp:66-72)
__device__ __forceinline__ uint32_t bucket_in_part(const Arith& a, uint64_t h) {
    return (uint32_t)__umul64hi(a.B, gamma_rt(a, a.P * h));
}
// slot within the part: reduce(y), the exact y mod S, or the pow2 form (reduce.hpp:67-72)
__device__ __forceinline__ uint32_t slot_of_y(const Arith& a, uint64_t y) {
    if (a.p2) return (uint32_t)(__umul64hi(kC, y) & (a.S - 1));
    if (a.mf.ok) return mod_fast(y, a.mf.S, a.mf.nS, a.mf.c, a.mf.m1, a.mf.m2);
    uint64_t r = y - __umul64hi(y, a.fm) * a.S;
    while (r >= a.S) r -= a.S;
    return (uint32_t)r;
}

struct Work {          // per-CTA workspace in global memory
    uint32_t* start;   // [B + 1] first hash of each bucket
    uint32_t* ord;     // [B]     bucket ids in visiting order (non-empty buckets)
    uint32_t* owner;   // [S]     bucket holding each slot
    uint64_t* hre;     // [max part size] the small buckets' hashes in visiting order
    unsigned long long* bigk;  // [B] heap keys of the buckets over kMaxK keys
    uint32_t* scratch; // [S] claim tags of a big bucket's eviction pricing (distinctness)
};

struct Shared {
    uint32_t cnt[kMaxK + 2];               // buckets per size
    uint32_t cbeg[kMaxK + 2];              // first visiting index of each size class
    uint32_t cpos[kMaxK + 2];              // first hre position of each size class
    uint32_t wbase[kSThreads / 32][kMaxK + 2];
    uint32_t wmin[kSThreads / 32];
    unsigned long long wkey[kSThreads / 32];
    unsigned long long costs[256];         // a big bucket's eviction cost per pilot
    uint32_t bad[8];                       // ... and the pilots ruled out
    uint32_t bsl[kSThreads / 32][kMaxK];   // batch mode: each warp's winning pilot's slots
    uint32_t bwin[kSThreads / 32];         //             its pilot (32 = none of the first 32)
    uint32_t bkc[kSThreads / 32];          //             its bucket's size
    uint32_t bsel[kSThreads / 32];         //             the warp that won each bucket
    uint32_t ncommit;
    uint32_t esl[kMaxK];                   // the evicting pilot's slots
    uint32_t recent[kRecent];
    unsigned long long heap[kHeapCap];
    uint32_t hn;
    uint32_t nbig;                         // buckets over kMaxK keys
    uint32_t flags;                        // 1 = part failed, 2 = unsupported
    uint32_t evictions;
    uint32_t by_pct[100];
    uint32_t part;
};

__device__ __forceinline__ unsigned long long bkey(uint32_t b, uint32_t sz) {
    return ((unsigned long long)sz << 32) | (0xffffffffu - b);  // engine.hpp:335 heap order
}
__device__ void heap_push(Shared& sm, unsigned long long k) {
    PH_SCHECK(sm.hn < kHeapCap);
    uint32_t i = sm.hn++;
    while (i) {
        const uint32_t p = (i - 1) >> 1;
        if (sm.heap[p] >= k) break;
        sm.heap[i] = sm.heap[p];
        i = p;
    }
    sm.heap[i] = k;
}
__device__ void heap_pop(Shared& sm) {
    PH_SCHECK(sm.hn >= 1 && sm.hn <= kHeapCap);
    const unsigned long long k = sm.heap[--sm.hn];
    uint32_t i = 0;
    for (;;) {
        uint32_t c = 2 * i + 1;
        if (c >= sm.hn) break;
        if (c + 1 < sm.hn && sm.heap[c + 1] > sm.heap[c]) c++;
        if (sm.heap[c] <= k) break;
        sm.heap[i] = sm.heap[c];
        i = c;
    }
    if (sm.hn) sm.heap[i] = k;
}

__device__ __forceinline__ bool distinct(const uint32_t* s, uint32_t k) {
    for (uint32_t i = 1; i < k; i++)
        for (uint32_t j = 0; j < i; j++)
            if (s[i] == s[j]) return false;
    return true;
}

// free_pilot's test of one pilot for a bucket of at most KB keys, the slots in registers
// (a per-thread array indexed at run time lives in local memory, and with ~210 KB of the SM's
// 256 KB carved out for the two CTAs' bitmaps the L1 cannot hold it: every read went to L2).
constexpr int kRegK = 8;
template <int KB>
__device__ __forceinline__ bool test_pilot_reg(const Arith& a, const uint32_t* taken,
                                               const uint64_t* kq, uint32_t kc, uint64_t hl,
                                               uint32_t (&r)[KB]) {
    uint32_t busy = 0;  // no early exit: the kc slot computations are independent chains
#pragma unroll
    for (int i = 0; i < KB; i++) {
        r[i] = 0xffffffffu - i;  // beyond kc: distinct dummies (slots are < 2^31)
        if (i < (int)kc) {
            r[i] = slot_of_y(a, kq[i] ^ hl);
            PH_SCHECK(r[i] < a.S);
            busy |= taken[r[i] >> 5] >> (r[i] & 31);
        }
    }
    bool ok = !(busy & 1);
    if (ok) {
#pragma unroll
        for (int i = 1; i < KB; i++)
#pragma unroll
            for (int j = 0; j < i; j++) ok &= r[i] != r[j];
    }
    return ok;
}

// Smallest lane of `cand` (lanes whose pilot's slots sl[0..k) are all free) whose slots are
// pairwise distinct, or 32: the candidate writes its slots to the warp's shared row and lane i
// compares slot i with the slots before it (O(k) per candidate instead of a k^2 loop over a
// local-memory array). Leaves the winner's slots in row[0..k). k <= 32.
__device__ __forceinline__ uint32_t first_distinct(unsigned cand, const uint32_t* sl, uint32_t k,
                                                   uint32_t* row, unsigned lane) {
    while (cand) {
        const uint32_t l0 = (uint32_t)__ffs(cand) - 1;
        if (lane == l0)
            for (uint32_t i = 0; i < k; i++) row[i] = sl[i];
        __syncwarp();
        bool dup = false;
        if (lane < k) {
            const uint32_t mine = row[lane];
            for (uint32_t j = 0; j < lane; j++) dup |= row[j] == mine;
        }
        const bool anyd = __any_sync(kFull, dup);
        __syncwarp();
        if (!anyd) return l0;
        cand &= cand - 1;
    }
    return 32;
}

// status[0]: a part failed (reseed); status[1]: unsupported shape (host search);
// status[2]: next part to claim; status[3]: total evictions; by_pct: 100 counters.
__device__ unsigned long long g_prof[16];  // cycles: prologue, batch steps, full steps; counts
__global__ void __launch_bounds__(kSThreads, 2) k_search_parts(
    const Arith a, const uint64_t* __restrict__ hashes, const uint64_t* __restrict__ off,
    uint8_t* __restrict__ pilots, uint32_t* __restrict__ taken_out, uint32_t words,
    Work* __restrict__ works, unsigned long long* __restrict__ status,
    unsigned long long* __restrict__ by_pct) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    Shared& sm = *reinterpret_cast<Shared*>(smem_raw);
    uint32_t* taken = reinterpret_cast<uint32_t*>(smem_raw + ((sizeof(Shared) + 15) & ~size_t{15}));
    const unsigned tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const Work w = works[blockIdx.x];
    const uint32_t S = (uint32_t)a.S, B = (uint32_t)a.B;
    const uint64_t hp = kC * ((uint64_t)tid ^ a.seed);  // hash_pilot(tid), hash.hpp:30-32
    uint32_t sl[kMaxK];

    for (;;) {
        __syncthreads();
        if (tid == 0) {
            const bool halt = *(volatile unsigned long long*)status || *(volatile unsigned long long*)(status + 1);
            sm.part = halt ? 0xffffffffu : (uint32_t)atomicAdd(status + 2, 1ull);
            sm.hn = 0;
            sm.nbig = 0;
            sm.flags = 0;
            sm.evictions = 0;
        }
        if (tid < 100) sm.by_pct[tid] = 0;
        if (tid < kRecent) sm.recent[tid] = kNoBucket;
        for (uint32_t i = tid; i < kMaxK + 2; i += kSThreads) sm.cnt[i] = 0;
        __syncthreads();
        const uint32_t part = sm.part;
        if (part >= a.P) break;
        const uint64_t* h = hashes + off[part];
        const uint32_t m = (uint32_t)(off[part + 1] - off[part]);
        uint8_t* pl = pilots + (uint64_t)part * B;

        // ---- prologue ------------------------------------------------------------------
        long long t_p0 = clock64(), t_batch = 0, t_full = 0, n_batch = 0, n_full = 0;
        for (uint32_t i = tid; i < words; i += kSThreads) taken[i] = 0;
        for (uint32_t i = tid; i < S; i += kSThreads) {
            w.owner[i] = kNoBucket;
            w.scratch[i] = 0;
        }
        for (uint32_t i = tid; i < B; i += kSThreads) pl[i] = 0;
        {   // bucket boundaries: thread t scans a contiguous chunk of the sorted hashes
            const uint32_t per = (m + kSThreads - 1) / kSThreads;
            const uint32_t i0 = min(m, tid * per), i1 = min(m, i0 + per);
            int64_t prev = i0 ? (int64_t)bucket_in_part(a, h[i0 - 1]) : -1;
            for (uint32_t i = i0; i < i1; i++) {
                const int64_t b = bucket_in_part(a, h[i]);
                for (int64_t q = prev + 1; q <= b; q++) w.start[q] = i;
                prev = b;
            }
            if (i1 == m && i0 < m) {  // the thread holding the last hash closes the table
                for (int64_t q = prev + 1; q <= (int64_t)B; q++) w.start[q] = m;
            }
            if (m == 0)
                for (uint32_t q = tid; q <= B; q += kSThreads) w.start[q] = 0;
        }
        __syncthreads();
        // sizes: per-warp ranges of bucket ids, so the counting sort below is stable
        const uint32_t wper = (B + kSThreads / 32 - 1) / (kSThreads / 32);
        const uint32_t b0 = min(B, warp * wper), b1 = min(B, b0 + wper);
        for (uint32_t s = lane; s < kMaxK + 2; s += 32) sm.wbase[warp][s] = 0;
        __syncwarp();
        for (uint32_t b = b0 + lane; b < b1; b += 32) {
            const uint32_t sz = __ldcg(w.start + b + 1) - __ldcg(w.start + b);
            if (sz > kMaxK) w.bigk[atomicAdd(&sm.nbig, 1u)] = bkey(b, sz);
            else atomicAdd(&sm.wbase[warp][sz], 1u);
        }
        __syncthreads();
        const uint32_t nbig = sm.nbig;
        // the big buckets lead the visiting order, by (size desc, id asc): rank sort
        for (uint32_t i = tid; i < nbig; i += kSThreads) {
            const unsigned long long ki = __ldcg(w.bigk + i);
            uint32_t rank = 0;
            for (uint32_t j = 0; j < nbig; j++) rank += __ldcg(w.bigk + j) > ki;
            PH_SCHECK(rank < nbig);
            w.ord[rank] = 0xffffffffu - (uint32_t)ki;
        }
        if (tid == 0) {  // class tables: sizes descending, within a size warps ascending
            uint32_t at = nbig, pos = 0;
            for (int s = kMaxK; s >= 1; s--) {
                uint32_t c = 0;
                sm.cbeg[s] = at;
                sm.cpos[s] = pos;
                for (int q = 0; q < kSThreads / 32; q++) {
                    const uint32_t x = sm.wbase[q][s];
                    sm.wbase[q][s] = at + c;
                    c += x;
                }
                sm.cnt[s] = c;
                at += c;
                pos += c * (uint32_t)s;
            }
            sm.cbeg[0] = at;  // = number of non-empty buckets
            sm.cnt[0] = 0;
        }
        __syncthreads();
        const uint32_t nonempty = sm.cbeg[0];
        // stable placement (ids ascending within a size) + the hashes in visiting order
        for (uint32_t bb = b0; bb < b1; bb += 32) {
            const uint32_t b = bb + lane;
            const uint32_t st = b < b1 ? __ldcg(w.start + b) : 0;
            uint32_t sz = b < b1 ? __ldcg(w.start + b + 1) - st : 0;
            if (sz > kMaxK) sz = 0;  // big buckets were placed by the rank sort above
            const unsigned mm = __match_any_sync(kFull, sz);
            const uint32_t rank = __popc(mm & ((1u << lane) - 1));
            uint32_t idx = 0;
            if (sz) idx = sm.wbase[warp][sz] + rank;
            __syncwarp();
            if (sz && rank == 0) sm.wbase[warp][sz] += __popc(mm);
            __syncwarp();
            if (sz) {
                PH_SCHECK(idx < nonempty && idx >= sm.cbeg[sz] && idx < sm.cbeg[sz] + sm.cnt[sz] &&
                          sm.cpos[sz] + (uint64_t)(idx - sm.cbeg[sz] + 1) * sz <= a.hre_cap);
                w.ord[idx] = b;
                uint64_t* dst = w.hre + sm.cpos[sz] + (uint64_t)(idx - sm.cbeg[sz]) * sz;
                for (uint32_t i = 0; i < sz; i++) dst[i] = h[st + i];
            }
        }
        __syncthreads();

        // ---- main loop -----------------------------------------------------------------
        const long long t_pro = clock64() - t_p0;
        uint32_t cursor = 0, kcur = kMaxK, rpos = 0, part_ev = 0, tag_base = 0;
        while (kcur > 1 && sm.cnt[kcur] == 0) kcur--;

        const uint64_t budget = 10ull * S;
        bool failed = false, single = false;
        uint32_t wpb = 1;  // batch mode: warps (x 32 pilots) per bucket
        uint32_t cend = 0;  // end of the current size class in the visiting order
        for (;;) {
            // next bucket: the larger of the heap's top and the visiting order's head
            const uint32_t hn = sm.hn;
            if (cursor == nonempty && hn == 0) break;
            if (cursor >= nbig && cursor < nonempty && cursor >= cend) {
                while (cursor >= sm.cbeg[kcur] + sm.cnt[kcur]) kcur--;
                cend = sm.cbeg[kcur] + sm.cnt[kcur];  // (kept in a register between steps)
            }
            if (!single && hn == 0 && cursor >= nbig && cursor < nonempty) {
                // Batch mode (no evicted bucket pending): the next eight buckets at once, one per
                // warp. A warp tests its bucket's pilots 32 at a time, smallest first, against
                // the bitmap as it stands, until one is free (eight rounds cover all 256). The
                // buckets commit in visiting order; a bucket commits if its pilot's slots are
                // still free after the earlier commits of the batch (bits are only set here, so
                // no smaller pilot can have become free: the choice is the sequential search's).
                // A bucket that lost a slot restarts the next batch; one with no free pilot at
                // all goes to the full step below (an eviction).
                const long long t_b0 = clock64();
                const uint32_t nb = min(8u / wpb, nonempty - cursor);
                const uint32_t q = warp / wpb, c = cursor + q;
                uint32_t kc = kcur, mybk = 0;
                if (q < nb) {
                    if (c >= cend)
                        while (c >= sm.cbeg[kc] + sm.cnt[kc]) kc--;
                    PH_SCHECK(c < nonempty && kc >= 1 && kc <= kMaxK && c >= sm.cbeg[kc] &&
                              sm.cpos[kc] + (uint64_t)(c - sm.cbeg[kc] + 1) * kc <= a.hre_cap);
                    mybk = w.ord[c];
                    PH_SCHECK(mybk < B);
                    const uint64_t* kq = w.hre + sm.cpos[kc] + (uint64_t)(c - sm.cbeg[kc]) * kc;
                    uint32_t win = 32, round = 0;
                    uint32_t r8[kRegK];
                    for (; round < 8; round++) {  // 32 pilots per round, smallest first
                    const uint32_t pil = round * 32 + lane;
                    const uint64_t hl = kC * ((uint64_t)pil ^ a.seed);
                    bool ok = true;
                    if (kc <= 2) {  // (warp-uniform: the bucket is the warp's)
                        uint32_t r2[2];
                        ok = test_pilot_reg<2>(a, taken, kq, kc, hl, r2);
                        r8[0] = r2[0], r8[1] = r2[1];
                    } else if (kc <= 4) {
                        uint32_t r4[4];
                        ok = test_pilot_reg<4>(a, taken, kq, kc, hl, r4);
#pragma unroll
                        for (int i = 0; i < 4; i++) r8[i] = r4[i];
                    } else if (kc <= kRegK) {
                        ok = test_pilot_reg<kRegK>(a, taken, kq, kc, hl, r8);
                    } else {
                        for (uint32_t i = 0; i < kc; i++) {
                            const uint32_t s1 = slot_of_y(a, kq[i] ^ hl);
                            if ((taken[s1 >> 5] >> (s1 & 31)) & 1) {
                                ok = false;
                                break;
                            }
                            sl[i] = s1;
                        }
                    }
                    const unsigned bal = __ballot_sync(kFull, ok);
                    if (kc <= kRegK) {
                        win = bal ? (uint32_t)__ffs(bal) - 1 : 32u;
                        if (lane == win) {
#pragma unroll
                            for (int i = 0; i < kRegK; i++)
                                if (i < (int)kc) sm.bsl[warp][i] = r8[i];
                        }
                    } else {
                        win = first_distinct(bal, sl, kc, sm.bsl[warp], lane);
                    }
                    if (win < 32) break;
                    }
                    if (lane == 0) {
                        sm.bwin[warp] = win < 32 ? round * 32 + win : 256u;
                        sm.bkc[warp] = kc;
                    }
                    if (tid == 0) {
                        asm volatile("prefetch.global.L2 [%0];" ::"l"(kq + 192));
                        asm volatile("prefetch.global.L2 [%0];" ::"l"(w.ord + cursor + 256));
                    }
                }
                __syncthreads();
                // Commit. Common case: every bucket up to the first one without a pilot
                // claims its slots at once (one atomicOr per slot); a claim that finds its bit
                // set lost the slot to another bucket of the batch, and then all claims are
                // rolled back and warp 0 commits the batch serially in visiting order.
                // lane x < 8 holds warp x's result; a segmented minimum over each bucket's wpb
                // warps gives every bucket's pilot and the warp holding it (pilot << 8 | warp)
                uint32_t pv = lane < 8 && lane / wpb < nb ? sm.bwin[lane] << 8 | lane : 256u << 8 | (lane & 7);
                for (uint32_t o = 1; o < wpb; o <<= 1) pv = min(pv, __shfl_xor_sync(kFull, pv, o));
                const unsigned lead = lane < 8 && lane % wpb == 0 && lane / wpb < nb;  // one lane per bucket
                const unsigned none = __ballot_sync(kFull, lead && (pv >> 8) == 256);
                const uint32_t nf = none ? ((uint32_t)__ffs(none) - 1) / wpb : nb;
                const unsigned high = __ballot_sync(kFull, lead && lane / wpb < nf && (pv >> 8) >= 16 * wpb);
                const uint32_t mybw = __shfl_sync(kFull, pv, (q * wpb) & 7) & 0xff;
                if (warp == 0 && lead && lane / wpb < nf) sm.bsel[lane / wpb] = pv & 0xff;
                bool hit = false, claimed = false;
                uint32_t s2 = 0;
                if (q < nf && warp == mybw && lane < kc) {
                    s2 = sm.bsl[warp][lane];
                    PH_SCHECK(s2 < S && mybw < kSThreads / 32);
                    hit = (atomicOr(&taken[s2 >> 5], 1u << (s2 & 31)) >> (s2 & 31)) & 1;
                    claimed = !hit;
                }
                if (tid == 0) {
                    sm.ncommit = nf | (nf < nb ? 1u : 0u) << 8 | (!high ? 1u << 16 : 0);
                    if (((cursor + nf) & 4095) < nf && *(volatile unsigned long long*)status) sm.flags |= 1;
                }
                const int anyhit = __syncthreads_or(hit);
                if (anyhit) {
                    if (claimed) atomicAnd(&taken[s2 >> 5], ~(1u << (s2 & 31)));
                    __syncthreads();
                if (warp == 0) {
                    uint32_t nc = 0, maxwin = 0, why = 0;  // why: 1 = no pilot, 2 = lost a slot
                    for (; nc < nb; nc++) {
                        uint32_t bw = nc * wpb;  // the bucket's warp holding the smallest pilot
                        for (uint32_t x = 1; x < wpb; x++)
                            if (sm.bwin[nc * wpb + x] < sm.bwin[bw]) bw = nc * wpb + x;
                        const uint32_t pw = sm.bwin[bw], kq = sm.bkc[bw];
                        if (pw == 256) {
                            why = 1;
                            break;
                        }
                        const uint32_t s1 = lane < kq ? sm.bsl[bw][lane] : 0;
                        const bool hit = lane < kq && ((taken[s1 >> 5] >> (s1 & 31)) & 1);
                        if (__any_sync(kFull, hit)) {
                            why = 2;
                            break;
                        }
                        if (lane < kq) atomicOr(&taken[s1 >> 5], 1u << (s1 & 31));
                        __syncwarp();
                        maxwin = max(maxwin, pw);
                        if (lane == 0) sm.bsel[nc] = bw;
                    }
                    if (lane == 0) {
                        sm.ncommit = nc | why << 8 | (maxwin < 16 * wpb ? 1u << 16 : 0);
                        if (((cursor + nc) & 4095) < nc && *(volatile unsigned long long*)status) sm.flags |= 1;
                    }
                }
                __syncthreads();
                }
                const uint32_t nc = sm.ncommit & 0xff, why = (sm.ncommit >> 8) & 0xff;
                if (q < nc && sm.bsel[q] == warp) {  // the winning warp publishes
                    if (lane < kc) w.owner[sm.bsl[warp][lane]] = mybk;
                    if (lane == 0) pl[mybk] = (uint8_t)sm.bwin[warp];
                }
                cursor += nc;
                if (why == 1) single = true;  // none of the 256 pilots is free: an eviction
                if (sm.flags) {
                    failed = true;
                    break;
                }
                t_batch += clock64() - t_b0;
                n_batch++;
                continue;
            }
            single = false;
            const long long t_f0 = clock64();
            n_full++;
            uint32_t bk = 0, k = 0;
            const uint64_t* kh;
            bool from_heap = false;
            if (cursor < nonempty) {
                bk = w.ord[cursor];
                k = cursor < nbig ? __ldcg(w.start + bk + 1) - __ldcg(w.start + bk) : kcur;
            }
            if (hn && (cursor == nonempty || sm.heap[0] > bkey(bk, k))) from_heap = true;
            if (from_heap) {
                bk = 0xffffffffu - (uint32_t)sm.heap[0];
                PH_SCHECK(bk < B);
                const uint32_t st = __ldcg(w.start + bk);
                k = __ldcg(w.start + bk + 1) - st;
                kh = h + st;
            } else if (cursor < nbig) {
                kh = h + __ldcg(w.start + bk);
            } else {
                kh = w.hre + sm.cpos[k] + (uint64_t)(cursor - sm.cbeg[k]) * k;
                if (tid == 0) {  // the stream a few buckets ahead into L1/L2
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(kh + 96));
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(w.ord + cursor + 96));
                }
            }
            if (k > kMaxK) {
                // A big bucket: the CTA tests one pilot at a time, keys across the threads;
                // free_pilot's two conditions (engine.hpp:131-147) are "no slot taken" (a
                // read-only pass) and "pairwise distinct" (every key claims its bit: a bit
                // already set is a self-collision, and the claims are rolled back).
                uint32_t p = 0;
                for (; p < 256; p++) {
                    const uint64_t hpp = kC * ((uint64_t)p ^ a.seed);
                    bool bad = false;
                    for (uint32_t i = tid; i < k && !bad; i += kSThreads) {
                        const uint32_t s = slot_of_y(a, kh[i] ^ hpp);
                        bad = (taken[s >> 5] >> (s & 31)) & 1;
                    }
                    if (__syncthreads_or(bad)) continue;
                    bool dup = false;
                    for (uint32_t i = tid; i < k; i += kSThreads) {
                        const uint32_t s = slot_of_y(a, kh[i] ^ hpp);
                        dup |= (atomicOr(&taken[s >> 5], 1u << (s & 31)) >> (s & 31)) & 1;
                    }
                    if (!__syncthreads_or(dup)) break;
                    for (uint32_t i = tid; i < k; i += kSThreads) {
                        const uint32_t s = slot_of_y(a, kh[i] ^ hpp);
                        atomicAnd(&taken[s >> 5], ~(1u << (s & 31)));
                    }
                    __syncthreads();
                }
                if (p == 256) {
                    // cheapest_pilot (engine.hpp:149-178) for a big bucket: all (pilot, key)
                    // pairs across the threads. Distinctness by claiming scratch[slot] with a
                    // tag unique to (this eviction, pilot): reading the tag back is a
                    // self-collision. Costs and disqualifications accumulate per pilot.
                    sm.costs[tid] = 0;
                    if (tid < 8) sm.bad[tid] = 0;
                    tag_base += 256;  // (2^24 big evictions per part before tags could repeat)
                    __syncthreads();
                    for (uint32_t q = 0; q < 256; q++) {
                        const uint64_t hq = kC * ((uint64_t)q ^ a.seed);
                        unsigned long long cost = 0;
                        bool out = false;
                        for (uint32_t i = tid; i < k; i += kSThreads) {
                            const uint32_t s = slot_of_y(a, kh[i] ^ hq);
                            out |= atomicExch(w.scratch + s, tag_base + q) == tag_base + q;
                            const uint32_t o = __ldcg(w.owner + s);
                            if (o == kNoBucket) continue;
#pragma unroll
                            for (int r = 0; r < kRecent; r++) out |= sm.recent[r] == o;
                            const unsigned long long sz = __ldcg(w.start + o + 1) - __ldcg(w.start + o);
                            cost += sz * sz;
                        }
                        if (cost) atomicAdd(&sm.costs[q], cost);
                        if (out) atomicOr(&sm.bad[q >> 5], 1u << (q & 31));
                        __syncthreads();  // pilot q's claims are complete before q + 1 overwrites them
                    }
                    unsigned long long key = (sm.bad[tid >> 5] >> (tid & 31)) & 1 ? ~0ull : sm.costs[tid] << 9 | tid;
#pragma unroll
                    for (int o = 16; o; o >>= 1) {
                        const unsigned long long y = __shfl_xor_sync(kFull, key, o);
                        key = y < key ? y : key;
                    }
                    if (lane == 0) sm.wkey[warp] = key;
                    __syncthreads();
                    key = sm.wkey[0];
#pragma unroll
                    for (int q = 1; q < kSThreads / 32; q++) key = sm.wkey[q] < key ? sm.wkey[q] : key;
                    if (key == ~0ull) {
                        if (tid == 0) sm.flags |= 1;  // no pilot is distinct and clear of recent buckets
                    } else if (tid == 0) {
                        const uint32_t ps = (uint32_t)(key & 511);
                        const uint64_t hs = kC * ((uint64_t)ps ^ a.seed);
                        if (from_heap) heap_pop(sm);
                        pl[bk] = (uint8_t)ps;
                        for (uint32_t i = 0; i < k; i++) {
                            const uint32_t s = slot_of_y(a, kh[i] ^ hs);
                            const uint32_t v = __ldcg(w.owner + s);
                            if (v != kNoBucket) {  // displace v entirely
                                const uint64_t vhp = kC * ((uint64_t)__ldcg(pl + v) ^ a.seed);
                                const uint32_t v0 = __ldcg(w.start + v), v1 = __ldcg(w.start + v + 1);
                                for (uint32_t j = v0; j < v1; j++) {
                                    const uint32_t vs = slot_of_y(a, h[j] ^ vhp);
                                    taken[vs >> 5] &= ~(1u << (vs & 31));
                                    __stcg(w.owner + vs, kNoBucket);
                                }
                                if (sm.hn >= kHeapCap) {
                                    sm.flags |= 2;
                                    break;
                                }
                                heap_push(sm, bkey(v, v1 - v0));
                                part_ev++;
                                sm.evictions++;
                                const uint64_t pct = (uint64_t)cursor * 100 / (nonempty ? nonempty : 1);
                                sm.by_pct[pct < 99 ? pct : 99]++;
                                if (part_ev > budget) sm.flags |= 1;
                            }
                            taken[s >> 5] |= 1u << (s & 31);
                            __stcg(w.owner + s, bk);
                        }
                        sm.recent[rpos] = bk;
                    }
                    rpos = (rpos + 1) % kRecent;
                } else {
                    for (uint32_t i = tid; i < k; i += kSThreads)
                        w.owner[slot_of_y(a, kh[i] ^ (kC * ((uint64_t)p ^ a.seed)))] = bk;
                    if (tid == 0) {
                        pl[bk] = (uint8_t)p;
                        if (from_heap) heap_pop(sm);
                    }
                }
                if (!from_heap) cursor++;
                __syncthreads();
                if (sm.flags) {
                    failed = (sm.flags & 1) != 0;
                    break;
                }
                continue;
            }
            // free_pilot (engine.hpp:131-147): thread p tests pilot p
            bool ok = true;
            if (k <= kRegK) {
                uint32_t r8[kRegK];
                ok = test_pilot_reg<kRegK>(a, taken, kh, k, hp, r8);
                if (ok) {
#pragma unroll
                    for (int i = 0; i < kRegK; i++) sl[i] = r8[i];
                }
            } else {
                for (uint32_t i = 0; i < k; i++) {
                    const uint32_t s = slot_of_y(a, kh[i] ^ hp);
                    if ((taken[s >> 5] >> (s & 31)) & 1) {
                        ok = false;
                        break;
                    }
                    sl[i] = s;
                }
            }
            unsigned bal = __ballot_sync(kFull, ok);
            if (k > kRegK) {
                const uint32_t l0 = first_distinct(bal, sl, k, sm.bsl[warp], lane);
                bal = l0 < 32 ? 1u << l0 : 0u;
            }
            if (lane == 0) sm.wmin[warp] = bal ? warp * 32 + (__ffs(bal) - 1) : 256u;
            __syncthreads();  // B1 (every thread has read the heap's top)
            uint32_t pstar = 256;
#pragma unroll
            for (int q = 0; q < kSThreads / 32; q++) pstar = min(pstar, sm.wmin[q]);
            if (pstar < 256) {
                if (tid == pstar) {
                    for (uint32_t i = 0; i < k; i++) {
                        PH_SCHECK(sl[i] < S && bk < B);
                        taken[sl[i] >> 5] |= 1u << (sl[i] & 31);
                        w.owner[sl[i]] = bk;
                    }
                    pl[bk] = (uint8_t)pstar;
                    if (from_heap) heap_pop(sm);
                }
            } else {
                // cheapest_pilot (engine.hpp:149-178): least total squared size of the
                // displaced buckets, never a recent displacer; ties to the smaller pilot
                unsigned long long key = ~0ull;
                for (uint32_t i = 0; i < k; i++) sl[i] = slot_of_y(a, kh[i] ^ hp);
                if (distinct(sl, k)) {
                    unsigned long long cost = 0;
                    bool good = true;
                    for (uint32_t i = 0; i < k && good; i++) {
                        const uint32_t o = __ldcg(w.owner + sl[i]);
                        if (o == kNoBucket) continue;
#pragma unroll
                        for (int r = 0; r < kRecent; r++) good &= sm.recent[r] != o;
                        const unsigned long long sz = __ldcg(w.start + o + 1) - __ldcg(w.start + o);
                        cost += sz * sz;
                    }
                    if (good) key = cost << 9 | tid;
                }
#pragma unroll
                for (int o = 16; o; o >>= 1) {
                    const unsigned long long y = __shfl_xor_sync(kFull, key, o);
                    key = y < key ? y : key;
                }
                if (lane == 0) sm.wkey[warp] = key;
                __syncthreads();
                key = sm.wkey[0];
#pragma unroll
                for (int q = 1; q < kSThreads / 32; q++) key = sm.wkey[q] < key ? sm.wkey[q] : key;
                if (key == ~0ull) {  // every pilot self-collides or hits a recent bucket
                    failed = true;
                    break;
                }
                pstar = (uint32_t)(key & 511);
                if (tid == pstar)
                    for (uint32_t i = 0; i < k; i++) sm.esl[i] = sl[i];
                __syncthreads();
                if (tid == 0) {
                    if (from_heap) heap_pop(sm);
                    pl[bk] = (uint8_t)pstar;
                    for (uint32_t i = 0; i < k; i++) {
                        const uint32_t s = sm.esl[i];
                        const uint32_t v = __ldcg(w.owner + s);
                        if (v != kNoBucket) {  // displace v entirely
                            const uint64_t vhp = kC * ((uint64_t)__ldcg(pl + v) ^ a.seed);
                            const uint32_t v0 = __ldcg(w.start + v), v1 = __ldcg(w.start + v + 1);
                            PH_SCHECK(v < B && v0 <= v1 && v1 <= m);
                            for (uint32_t j = v0; j < v1; j++) {
                                const uint32_t vs = slot_of_y(a, h[j] ^ vhp);
                                PH_SCHECK(vs < S && ((taken[vs >> 5] >> (vs & 31)) & 1));  // v held it
                                taken[vs >> 5] &= ~(1u << (vs & 31));
                                __stcg(w.owner + vs, kNoBucket);
                            }
                            if (sm.hn >= kHeapCap) {
                                sm.flags |= 2;
                                break;
                            }
                            heap_push(sm, bkey(v, v1 - v0));
                            part_ev++;
                            sm.evictions++;
                            // the reference's placed_first (buckets placed for the first
                            // time in earlier steps) == buckets taken from the order so far
                            const uint64_t pct = (uint64_t)cursor * 100 / (nonempty ? nonempty : 1);
                            sm.by_pct[pct < 99 ? pct : 99]++;
                            if (part_ev > budget) sm.flags |= 1;
                        }
                        taken[s >> 5] |= 1u << (s & 31);
                        __stcg(w.owner + s, bk);
                    }
                    sm.recent[rpos] = bk;
                }
                rpos = (rpos + 1) % kRecent;
            }
            t_full += clock64() - t_f0;
            if (!from_heap) cursor++;
            if (tid == 0 && (cursor & 1023) == 0 && !from_heap && *(volatile unsigned long long*)status)
                sm.flags |= 1;  // another part failed: the attempt is over
            __syncthreads();  // B2: bitmap, owner[], heap and flags of this step visible
            if (sm.flags) {
                failed = (sm.flags & 1) != 0;
                break;
            }
        }
        if (sm.flags & 2) {
            if (tid == 0) atomicExch(status + 1, 1ull);
            break;
        }
        if (failed) {
            if (tid == 0) atomicExch(status, 1ull);
            break;
        }
        // ---- epilogue: the part's occupancy bitmap and statistics ----------------------
        uint32_t* to = taken_out + (uint64_t)part * words;
        for (uint32_t i = tid; i < words; i += kSThreads) to[i] = taken[i];
        if (tid == 0) {
            atomicAdd(g_prof + 0, (unsigned long long)t_pro);
            atomicAdd(g_prof + 1, (unsigned long long)t_batch);
            atomicAdd(g_prof + 2, (unsigned long long)t_full);
            atomicAdd(g_prof + 3, (unsigned long long)n_batch);
            atomicAdd(g_prof + 4, (unsigned long long)n_full);
            atomicAdd(g_prof + 5, 1ull);
        }
        if (tid == 0 && sm.evictions) atomicAdd(status + 3, (unsigned long long)sm.evictions);
        if (tid < 100 && sm.by_pct[tid]) atomicAdd(by_pct + tid, (unsigned long long)sm.by_pct[tid]);
    }
}

}  // namespace

// Violations counted by a checked build's search kernel since the last call; -1 otherwise.
int search_check_errors(uint64_t* count, uint64_t* line) {
#ifdef PH_CHECKS
    unsigned long long h[2] = {0, 0};
    if (cudaMemcpyFromSymbol(h, g_schk, sizeof(h)) != cudaSuccess) return -2;
    const unsigned long long z[2] = {0, 0};
    cudaMemcpyToSymbol(g_schk, z, sizeof(z));
    *count = h[0];
    *line = h[1];
    return 0;
#else
    *count = *line = 0;
    return -1;
#endif
}

size_t search_smem_bytes(uint64_t S) {
    return ((sizeof(Shared) + 15) & ~size_t{15}) + ((S + 31) / 32) * 4;
}

// Can the kernel take this shape? The occupancy bitmap must fit in one CTA's shared memory
// (S <= ~1.7 M slots per part; up to ~830 k, config 3's 762 k included, two CTAs share an SM).
bool search_parts_supported(uint64_t S, uint64_t B, uint64_t max_part) {
    return S >= 1 && S < (1ull << 31) && B < (1ull << 31) && max_part < (1ull << 31) &&
           search_smem_bytes(S) <= 216 * 1024;
}

// Searches every part. d_hashes / d_off: build_prepare_u64's output. d_pilots: P*B bytes.
// d_taken: P * ceil(S/32) words. h_status[4] (see the kernel), h_by_pct[100]. Synchronous.
cudaError_t search_parts_gpu(const uint64_t* d_hashes, const uint64_t* d_off, uint64_t n, uint64_t P,
                             uint64_t S, uint64_t B, uint64_t seed, int fn, const uint64_t* d_opt,
                             uint64_t max_part, uint8_t* d_pilots, uint32_t* d_taken,
                             unsigned long long* h_status, unsigned long long* h_by_pct,
                             cudaStream_t s, int sms) {
    (void)n;
    Arith a{};
    a.P = P, a.S = S, a.B = B, a.seed = seed;
    a.p2 = (S & (S - 1)) == 0;
    a.fm = a.p2 ? 0 : ~0ull / S;
    a.opt = d_opt;
    a.fn = fn;
    a.mf = mod_fast_make(S);
    if (a.p2) a.mf.ok = false;
    a.hre_cap = max_part + 128;
    const uint32_t words = (uint32_t)((S + 31) / 32);
    const size_t smem = search_smem_bytes(S);
    cudaError_t e = cudaFuncSetAttribute(k_search_parts, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int bps = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_search_parts, kSThreads, smem);
    if (e != cudaSuccess) return e;
    if (bps < 1) return cudaErrorInvalidConfiguration;
    const int grid = (int)std::min<uint64_t>(P, (uint64_t)sms * bps);
    // per-CTA workspaces in one allocation
    const size_t w_start = ((B + 1) * 4 + 255) & ~size_t{255}, w_ord = (B * 4 + 255) & ~size_t{255};
    const size_t w_owner = (S * 4 + 255) & ~size_t{255}, w_hre = ((max_part + 128) * 8 + 255) & ~size_t{255};
    const size_t w_big = (B * 8 + 255) & ~size_t{255};
    const size_t per = w_start + w_ord + 2 * w_owner + w_hre + w_big;
    uint8_t* ws = nullptr;
    Work* d_works = nullptr;
    unsigned long long* d_status = nullptr;
    auto cleanup = [&] {
        if (ws) cudaFree(ws);
        if (d_works) cudaFree(d_works);
        if (d_status) cudaFree(d_status);
    };
    if ((e = cudaMalloc(&ws, per * grid)) != cudaSuccess || (e = cudaMalloc(&d_works, sizeof(Work) * grid)) != cudaSuccess ||
        (e = cudaMalloc(&d_status, (4 + 100) * 8)) != cudaSuccess) {
        cleanup();
        return e;
    }
    std::vector<Work> hw(grid);
    for (int i = 0; i < grid; i++) {
        uint8_t* b = ws + per * i;
        hw[i].start = reinterpret_cast<uint32_t*>(b);
        hw[i].ord = reinterpret_cast<uint32_t*>(b + w_start);
        hw[i].owner = reinterpret_cast<uint32_t*>(b + w_start + w_ord);
        hw[i].hre = reinterpret_cast<uint64_t*>(b + w_start + w_ord + w_owner);
        hw[i].bigk = reinterpret_cast<unsigned long long*>(b + w_start + w_ord + w_owner + w_hre);
        hw[i].scratch = reinterpret_cast<uint32_t*>(b + w_start + w_ord + w_owner + w_hre + w_big);
    }
    e = cudaMemcpyAsync(d_works, hw.data(), sizeof(Work) * grid, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(d_status, 0, (4 + 100) * 8, s);
    const bool trace = std::getenv("PH_GPU_BUILD_TRACE") != nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    if (trace) {
        unsigned long long z[16] = {};
        cudaMemcpyToSymbol(g_prof, z, sizeof(z));
        cudaEventCreate(&ev0);
        cudaEventCreate(&ev1);
        cudaEventRecord(ev0, s);
    }
    if (e == cudaSuccess) {
        k_search_parts<<<grid, kSThreads, smem, s>>>(a, d_hashes, d_off, d_pilots, d_taken, words, d_works,
                                                     d_status, d_status + 4);
        note_launch();
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(h_status, d_status, 4 * 8, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(h_by_pct, d_status + 4, 100 * 8, cudaMemcpyDeviceToHost, s);
    if (trace) cudaEventRecord(ev1, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (trace && e == cudaSuccess) {
        float ms = 0;
        cudaEventElapsedTime(&ms, ev0, ev1);
        unsigned long long pr[16] = {};
        cudaMemcpyFromSymbol(pr, g_prof, sizeof(pr));
        const double parts = pr[5] ? (double)pr[5] : 1.0;
        std::fprintf(stderr, "[ph_gpu search] kernel %.1f ms, grid %d; per part: prologue %.0f kcyc, batch steps "
                     "%.0f (%.0f kcyc), full steps %.0f (%.0f kcyc)\n", ms, grid, pr[0] / parts / 1e3,
                     pr[3] / parts, pr[1] / parts / 1e3, pr[4] / parts, pr[2] / parts / 1e3);
        cudaEventDestroy(ev0);
        cudaEventDestroy(ev1);
    }
    cleanup();
    return e;
}

}  // namespace phg
