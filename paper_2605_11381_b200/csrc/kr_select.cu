// kr_select.cu -- step 3 of the decision core: priority ordering and top-k
// batch admission under the edge budget (scheduler.py:130-140, 193-241).
//
// The reference sorts every pending request (Python `sorted`, bucket by
// bucket) and slices the first k = capacity - in_flight as the edge batch.  On
// the device the order is the ascending order of unique 128-bit keys
// (kr_urgency), so admission is:
//   1. MSD radix select of the k-th smallest key: each level histograms an
//      11-bit digit taken just below the highest bit on which the surviving
//      candidates still differ (OR ^ AND of the set), keeps only the boundary
//      bin, and stops when the boundary bin holds one key.  Two grid-wide levels
//      shrink 2^20 keys to a handful; one CTA finishes.
//   2. One elementwise admission pass (key <= kth): admitted / refetch masks,
//      skip counters (scheduler.py:223-234) and a block-aggregated gather of
//      the k admitted (key, index) pairs.
//   3. A sort of only those k pairs, independent of the key distribution:
//      runs of 1024 bitonic-sorted in shared memory, then every pair's final
//      position = its run index + binary-search ranks in the other runs
//      (k <= 2^17; beyond, a stable multi-CTA LSD radix sort over the
//      differing key bits), giving S_e in reference order.
// Keys are unique (the lexrank tiebreak), so every step is deterministic.
#include <atomic>
#include <climits>

#include "kr_common.cuh"
#include "kr_host.cuh"

namespace kr {

constexpr int kDigitBits = 11;
constexpr int kBins = 1 << kDigitBits;
#ifndef KR_SORT_TILE
#define KR_SORT_TILE 4096
#endif
constexpr int kSortTile = KR_SORT_TILE;  // LSD radix: elements per CTA tile (256 threads x 16)

struct SelState {
    unsigned long long st[2][4];  // [parity] {or_hi, or_lo, and_hi, and_lo}
    unsigned int cnt[2];          // [parity] candidate count
    long long need;               // 1-based rank of the target within candidates
    unsigned int dstar;
    unsigned int dcount;          // population of the boundary bin
    int done;
    int pad_;
    kr_key kth;
    unsigned int sel_count;       // admission gather count
    unsigned int pad2_[3];
    unsigned long long sst[4];    // OR/AND of the gathered (admitted) keys
    unsigned int hist[kBins];
};

struct Workspace {
    SelState* state;
    kr_key* cand[2];
    kr_key* skeys[2];
    int32_t* sidx[2];
    uint32_t* tile_hist;
};

static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

static size_t sort_tiles(int64_t n) { return static_cast<size_t>((n + kSortTile - 1) / kSortTile); }

static size_t workspace_bytes(int64_t n) {
    size_t nn = static_cast<size_t>(n < 1 ? 1 : n);
    size_t b = align256(sizeof(SelState));
    b += 2 * align256(nn * sizeof(kr_key));      // select candidates
    b += 2 * align256(nn * sizeof(kr_key));      // sort keys ping-pong
    b += 2 * align256(nn * sizeof(int32_t));     // sort index ping-pong
    b += align256(sort_tiles(n) * 256 * sizeof(uint32_t));
    return b;
}

static Workspace carve(void* ws, int64_t n) {
    size_t nn = static_cast<size_t>(n < 1 ? 1 : n);
    unsigned char* p = static_cast<unsigned char*>(ws);
    Workspace w;
    w.state = reinterpret_cast<SelState*>(p);
    p += align256(sizeof(SelState));
    for (int i = 0; i < 2; i++) {
        w.cand[i] = reinterpret_cast<kr_key*>(p);
        p += align256(nn * sizeof(kr_key));
    }
    for (int i = 0; i < 2; i++) {
        w.skeys[i] = reinterpret_cast<kr_key*>(p);
        p += align256(nn * sizeof(kr_key));
    }
    for (int i = 0; i < 2; i++) {
        w.sidx[i] = reinterpret_cast<int32_t*>(p);
        p += align256(nn * sizeof(int32_t));
    }
    w.tile_hist = reinterpret_cast<uint32_t*>(p);
    return w;
}

// ---------------------------------------------------------------------------
// block-level helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long warp_or(unsigned long long v) {
    for (int o = 16; o; o >>= 1) v |= __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ unsigned long long warp_and(unsigned long long v) {
    for (int o = 16; o; o >>= 1) v &= __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// OR / AND of keys: warp shuffles, then shared memory, then one set of
// global atomics per block (only if the block saw any key).
__device__ __forceinline__ void stats_accumulate(unsigned long long* dst, unsigned long long ohi,
                                                 unsigned long long olo, unsigned long long ahi,
                                                 unsigned long long alo) {
    __shared__ unsigned long long red[4][32];
    ohi = warp_or(ohi);
    olo = warp_or(olo);
    ahi = warp_and(ahi);
    alo = warp_and(alo);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = (blockDim.x + 31) >> 5;
    if (lane == 0) {
        red[0][warp] = ohi; red[1][warp] = olo; red[2][warp] = ahi; red[3][warp] = alo;
    }
    __syncthreads();
    if (warp == 0) {
        unsigned long long a = lane < nw ? red[0][lane] : 0ull;
        unsigned long long b = lane < nw ? red[1][lane] : 0ull;
        unsigned long long c = lane < nw ? red[2][lane] : ~0ull;
        unsigned long long d = lane < nw ? red[3][lane] : ~0ull;
        a = warp_or(a); b = warp_or(b); c = warp_and(c); d = warp_and(d);
        if (lane == 0 && (a | b | ~c | ~d)) {
            if (a) atomicOr(&dst[0], a);
            if (b) atomicOr(&dst[1], b);
            if (~c) atomicAnd(&dst[2], c);
            if (~d) atomicAnd(&dst[3], d);
        }
    }
}

// Block-aggregated append: returns this thread's slot (valid if `take`).
__device__ __forceinline__ unsigned block_append(bool take, unsigned int* counter) {
    __shared__ unsigned int wcnt[32];
    __shared__ unsigned int base;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = (blockDim.x + 31) >> 5;
    const unsigned ballot = __ballot_sync(0xffffffffu, take);
    if (lane == 0) wcnt[warp] = __popc(ballot);
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned total = 0;
        for (int w = 0; w < nw; w++) {
            unsigned c = wcnt[w];
            wcnt[w] = total;
            total += c;
        }
        base = total ? atomicAdd(counter, total) : 0u;
    }
    __syncthreads();
    const unsigned pos = base + wcnt[warp] + __popc(ballot & ((1u << lane) - 1));
    __syncthreads();  // wcnt / base reused by the next call
    return pos;
}

// Digit = the values of the candidate set's kDigitBits most significant
// *differing* bit positions (a pext of OR ^ AND), MSB first.  All candidates
// agree on every other bit, so digit order is key order; unlike a contiguous
// bit window it never wastes digit bits on constant fields (e.g. the high
// zero bits of the aged estimate between the bucket and its significant bits).
struct Digit {
    int W;                 // number of digit bits (0: all candidates identical)
    int nrun;              // the digit bits grouped into runs of adjacent positions
    int run_pos[kDigitBits];  // lowest bit position (0..127) of each run, MSB run first
    int run_len[kDigitBits];
    bool any;
};
// Built with compile-time indices only (predicated updates) so that the run
// table lives in registers for the per-key extraction loops.
__device__ __forceinline__ Digit digit_of(const unsigned long long* s) {
    unsigned long long xlo = s[1] ^ s[3], xhi = s[0] ^ s[2];
    Digit d;
    d.W = 0;
    d.nrun = 0;
#pragma unroll
    for (int r = 0; r < kDigitBits; r++) {
        d.run_pos[r] = 0;
        d.run_len[r] = 0;
    }
    int last = -2;
#pragma unroll
    for (int w = 0; w < kDigitBits; w++) {
        int pos = -1;
        if (xhi) {
            pos = 127 - __clzll(xhi);
            xhi &= ~(1ull << (pos - 64));
        } else if (xlo) {
            pos = 63 - __clzll(xlo);
            xlo &= ~(1ull << pos);
        }
        if (pos >= 0) {
            // extend the current run downwards unless it would cross the word boundary
            const bool extend = pos == last - 1 && (pos >> 6) == (last >> 6);
            const int cur = extend ? d.nrun - 1 : d.nrun;
#pragma unroll
            for (int r = 0; r < kDigitBits; r++) {
                if (r == cur) {
                    d.run_pos[r] = pos;
                    d.run_len[r] += 1;
                }
            }
            d.nrun = cur + 1;
            last = pos;
            d.W = w + 1;
        }
    }
    d.any = d.W > 0;
    return d;
}
__device__ __forceinline__ unsigned digit_val(const kr_key& k, const Digit& d) {
    unsigned v = 0;
#pragma unroll
    for (int r = 0; r < kDigitBits; r++) {
        if (r >= d.nrun) break;
        const int pos = d.run_pos[r], len = d.run_len[r];
        const unsigned long long word = pos >= 64 ? k.hi : k.lo;
        v = (v << len) | static_cast<unsigned>((word >> (pos & 63)) & ((1ull << len) - 1));
    }
    return v;
}

// ---------------------------------------------------------------------------
// radix select
// ---------------------------------------------------------------------------
__global__ void k_sel_reset(SelState* s, int64_t n, int64_t k, const unsigned long long* stats) {
    for (int i = threadIdx.x; i < kBins; i += blockDim.x) s->hist[i] = 0;
    if (threadIdx.x == 0) {
        for (int p = 0; p < 2; p++) {
            s->st[p][0] = 0; s->st[p][1] = 0; s->st[p][2] = ~0ull; s->st[p][3] = ~0ull;
        }
        if (stats)
            for (int j = 0; j < 4; j++) s->st[0][j] = stats[j];
        s->sst[0] = 0; s->sst[1] = 0; s->sst[2] = ~0ull; s->sst[3] = ~0ull;
        s->cnt[0] = static_cast<unsigned>(n);
        s->cnt[1] = 0;
        s->need = k;
        s->done = 0;
        s->sel_count = 0;
    }
}

__global__ void __launch_bounds__(256) k_sel_stats(const kr_key* __restrict__ keys, int64_t n,
                                                   SelState* s) {
    unsigned long long oh = 0, ol = 0, ah = ~0ull, al = ~0ull;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        kr_key k = keys[i];
        oh |= k.hi; ol |= k.lo; ah &= k.hi; al &= k.lo;
    }
    stats_accumulate(s->st[0], oh, ol, ah, al);
}

// level L reads candidates src (count cnt[L&1]) and histograms their digit.
__global__ void __launch_bounds__(256) k_sel_hist(const kr_key* __restrict__ src, SelState* s,
                                                  int level) {
    __shared__ unsigned int h[kBins];
    if (s->done) return;
    const int p = level & 1;
    Digit d = digit_of(s->st[p]);
    const int64_t n = s->cnt[p];
    const int bins = 1 << d.W;
    for (int i = threadIdx.x; i < bins; i += blockDim.x) h[i] = 0;
    __syncthreads();
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x)
        atomicAdd(&h[digit_val(src[i], d)], 1u);
    __syncthreads();
    for (int i = threadIdx.x; i < bins; i += blockDim.x)
        if (h[i]) atomicAdd(&s->hist[i], h[i]);
}

// One block: choose the boundary bin d* (cum_lt < need <= cum_le).
__device__ void sel_pick_block(SelState* s, int level, const unsigned int* hist,
                               const kr_key* src) {
    __shared__ unsigned int part[1024];
    __shared__ int found;
    const int p = level & 1;
    Digit d = digit_of(s->st[p]);
    if (!d.any) {  // all candidates identical: unique keys => a single one
        if (threadIdx.x == 0) {
            s->kth = src[0];
            s->done = 1;
        }
        return;
    }
    const int bins = 1 << d.W;
    const int per = (bins + blockDim.x - 1) / blockDim.x;
    unsigned int local = 0;
    for (int q = 0; q < per; q++) {
        int b = threadIdx.x * per + q;
        if (b < bins) local += hist[b];
    }
    part[threadIdx.x] = local;
    if (threadIdx.x == 0) found = 0;
    __syncthreads();
    // inclusive scan of part[] (Hillis-Steele)
    for (int o = 1; o < blockDim.x; o <<= 1) {
        unsigned int v = threadIdx.x >= o ? part[threadIdx.x - o] : 0;
        __syncthreads();
        part[threadIdx.x] += v;
        __syncthreads();
    }
    const long long need = s->need;
    unsigned long long before = threadIdx.x ? part[threadIdx.x - 1] : 0;
    if (static_cast<long long>(before) < need && need <= static_cast<long long>(part[threadIdx.x])) {
        unsigned long long cum = before;
        for (int q = 0; q < per; q++) {
            int b = threadIdx.x * per + q;
            if (b >= bins) break;
            unsigned int c = hist[b];
            if (static_cast<long long>(cum) < need && need <= static_cast<long long>(cum + c)) {
                s->dstar = static_cast<unsigned>(b);
                s->dcount = c;
                s->need = need - static_cast<long long>(cum);
                found = 1;
                break;
            }
            cum += c;
        }
    }
    __syncthreads();
    (void)found;
}

__global__ void __launch_bounds__(1024) k_sel_pick(SelState* s, const kr_key* src, int level) {
    if (s->done) return;
    sel_pick_block(s, level, s->hist, src);
    __syncthreads();
    // reset for the next level
    for (int i = threadIdx.x; i < kBins; i += blockDim.x) s->hist[i] = 0;
    if (threadIdx.x == 0) {
        const int q = (level + 1) & 1;
        s->st[q][0] = 0; s->st[q][1] = 0; s->st[q][2] = ~0ull; s->st[q][3] = ~0ull;
        s->cnt[q] = 0;
    }
}

// Keep the boundary bin; if it holds one key that key is the answer.
__global__ void __launch_bounds__(256) k_sel_scatter(const kr_key* __restrict__ src, kr_key* dst,
                                                     SelState* s, int level) {
    if (s->done) return;
    const int p = level & 1, q = (level + 1) & 1;
    Digit d = digit_of(s->st[p]);
    const int64_t n = s->cnt[p];
    const unsigned dstar = s->dstar;
    const bool single = s->dcount == 1;
    unsigned long long oh = 0, ol = 0, ah = ~0ull, al = ~0ull;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t base = blockIdx.x * int64_t(blockDim.x); base < n; base += stride) {
        int64_t i = base + threadIdx.x;
        bool keep = false;
        kr_key k{0, 0};
        if (i < n) {
            k = src[i];
            keep = digit_val(k, d) == dstar;
        }
        if (single) {
            if (keep) {
                s->kth = k;
                s->done = 1;
            }
            continue;
        }
        unsigned mask = __ballot_sync(0xffffffffu, keep);
        unsigned pos = 0;
        if (mask) {
            int lane = threadIdx.x & 31;
            int leader = __ffs(mask) - 1;
            unsigned basepos = 0;
            if (lane == leader) basepos = atomicAdd(&s->cnt[q], __popc(mask));
            basepos = __shfl_sync(0xffffffffu, basepos, leader);
            pos = basepos + __popc(mask & ((1u << lane) - 1));
        }
        if (keep) {
            dst[pos] = k;
            oh |= k.hi; ol |= k.lo; ah &= k.hi; al &= k.lo;
        }
    }
    if (!single) stats_accumulate(s->st[q], oh, ol, ah, al);
}

// Single CTA: remaining levels over global ping-pong buffers.
__global__ void __launch_bounds__(1024) k_sel_finish(SelState* s, kr_key* bufA, kr_key* bufB,
                                                     int level) {
    __shared__ unsigned int h[kBins];
    __shared__ unsigned long long sst[4];
    __shared__ unsigned int scnt;
    if (s->done) return;
    // bufA holds the candidates of `level` (the last grid-wide scatter's output)
    kr_key* src = bufA;
    kr_key* dst = bufB;
    int p = level & 1;
    for (int it = 0; it < 130; it++) {
        const unsigned n = s->cnt[p];
        Digit d = digit_of(s->st[p]);
        if (!d.any || n <= 1) {
            if (threadIdx.x == 0) {
                s->kth = src[0];
                s->done = 1;
            }
            return;
        }
        const int bins = 1 << d.W;
        for (int i = threadIdx.x; i < bins; i += blockDim.x) h[i] = 0;
        __syncthreads();
        for (unsigned i = threadIdx.x; i < n; i += blockDim.x) atomicAdd(&h[digit_val(src[i], d)], 1u);
        __syncthreads();
        sel_pick_block(s, p, h, src);
        __syncthreads();
        const unsigned dstar = s->dstar;
        const bool single = s->dcount == 1;
        if (threadIdx.x < 4) sst[threadIdx.x] = threadIdx.x < 2 ? 0ull : ~0ull;
        if (threadIdx.x == 0) scnt = 0;
        __syncthreads();
        unsigned long long oh = 0, ol = 0, ah = ~0ull, al = ~0ull;
        for (unsigned base = 0; base < n; base += blockDim.x) {
            unsigned i = base + threadIdx.x;
            bool keep = false;
            kr_key k{0, 0};
            if (i < n) {
                k = src[i];
                keep = digit_val(k, d) == dstar;
            }
            if (single) {
                if (keep) {
                    s->kth = k;
                    s->done = 1;
                }
                continue;
            }
            unsigned mask = __ballot_sync(0xffffffffu, keep);
            unsigned pos = 0;
            if (mask) {
                int lane = threadIdx.x & 31;
                int leader = __ffs(mask) - 1;
                unsigned bp = 0;
                if (lane == leader) bp = atomicAdd(&scnt, __popc(mask));
                bp = __shfl_sync(0xffffffffu, bp, leader);
                pos = bp + __popc(mask & ((1u << lane) - 1));
            }
            if (keep) {
                dst[pos] = k;
                oh |= k.hi; ol |= k.lo; ah &= k.hi; al &= k.lo;
            }
        }
        if (single) return;
        oh = warp_or(oh); ol = warp_or(ol); ah = warp_and(ah); al = warp_and(al);
        if ((threadIdx.x & 31) == 0) {
            atomicOr(&sst[0], oh); atomicOr(&sst[1], ol);
            atomicAnd(&sst[2], ah); atomicAnd(&sst[3], al);
        }
        __syncthreads();
        const int q = p ^ 1;
        if (threadIdx.x == 0) {
            s->st[q][0] = sst[0]; s->st[q][1] = sst[1]; s->st[q][2] = sst[2]; s->st[q][3] = sst[3];
            s->cnt[q] = scnt;
        }
        __syncthreads();
        p = q;
        kr_key* t = src; src = dst; dst = t;
    }
}

__global__ void k_set_key(kr_key* dst, unsigned long long hi, unsigned long long lo) {
    dst->hi = hi;
    dst->lo = lo;
}
__global__ void k_copy_kth(const SelState* s, kr_key* dst) { *dst = s->kth; }

// ---------------------------------------------------------------------------
// admission pass (scheduler.py:204-207, 223-234)
// ---------------------------------------------------------------------------
struct AdmitArgs {
    const kr_key* keys;
    int64_t n;
    int all;   // k >= n
    int none;  // k == 0
    const kr_key* kth;
    const int64_t* obs;     // nullable
    int32_t* skipped;       // nullable
    uint8_t* admitted;      // nullable
    uint8_t* refetch;       // nullable
    int64_t now, stale;
    kr_key* sel_keys;       // nullable (gather)
    int32_t* sel_idx;
    SelState* s;
};

__global__ void k_admit_init(SelState* s) {
    if (threadIdx.x == 0) {
        s->sel_count = 0;
        s->sst[0] = 0; s->sst[1] = 0; s->sst[2] = ~0ull; s->sst[3] = ~0ull;
    }
}

__global__ void __launch_bounds__(256) k_admit(AdmitArgs a) {
    kr_key kth{~0ull, ~0ull};
    if (!a.all && !a.none) kth = *a.kth;
    unsigned long long oh = 0, ol = 0, ah = ~0ull, al = ~0ull;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t base = blockIdx.x * int64_t(blockDim.x); base < a.n; base += stride) {
        int64_t i = base + threadIdx.x;
        bool in = false;
        kr_key k{0, 0};
        if (i < a.n) {
            k = a.keys[i];
            in = !a.none && (a.all || key_le(k, kth));
            if (a.admitted) a.admitted[i] = in;
            if (a.refetch) a.refetch[i] = in && (a.now - __ldg(a.obs + i) > a.stale);
            if (a.skipped) a.skipped[i] = in ? 0 : a.skipped[i] + 1;
        }
        if (a.sel_keys && __syncthreads_or(in)) {
            unsigned pos = block_append(in, &a.s->sel_count);
            if (in) {
                a.sel_keys[pos] = k;
                a.sel_idx[pos] = static_cast<int32_t>(i);
                oh |= k.hi; ol |= k.lo; ah &= k.hi; al &= k.lo;
            }
        }
    }
    if (a.sel_keys) stats_accumulate(a.s->sst, oh, ol, ah, al);
}

constexpr int kRun = 256;          // run length sorted in shared memory
constexpr int kRunThreads = 128;
constexpr int kRunSortMax = 1 << 17;  // larger sets use the multi-CTA LSD radix sort

__device__ __forceinline__ bool pair_gt(const kr_key& a, int32_t ia, const kr_key& b, int32_t ib) {
    if (a.hi != b.hi) return a.hi > b.hi;
    if (a.lo != b.lo) return a.lo > b.lo;
    return ia > ib;
}

// Sort of m (key, index) pairs, independent of the key distribution:
//  (1) each CTA sorts one run of kRun pairs with a bitonic network in shared
//      memory (padded with +inf);
//  (2) every pair's final position = its index inside its run + the number of
//      smaller pairs in every other run (binary search), computed by one thread
//      per pair and scattered directly.  Pairs are unique (index tiebreak), so
//      positions form a permutation.
struct Pair {
    kr_key k;
    int32_t i;
};

__device__ __forceinline__ Pair shfl_pair(const Pair& p, int lane_mask) {
    Pair q;
    q.k.hi = __shfl_xor_sync(0xffffffffu, p.k.hi, lane_mask);
    q.k.lo = __shfl_xor_sync(0xffffffffu, p.k.lo, lane_mask);
    q.i = __shfl_xor_sync(0xffffffffu, p.i, lane_mask);
    return q;
}

// keep the smaller pair of (mine, other) when keep_min, else the larger
__device__ __forceinline__ Pair keep(const Pair& mine, const Pair& other, bool keep_min) {
    const bool gt = pair_gt(mine.k, mine.i, other.k, other.i);
    return (gt == keep_min) ? other : mine;
}

// One run of kRun = 256 pairs per CTA, a bitonic network held in registers:
// thread t owns elements 2t and 2t + 1; partners at distance j = 1 are in the
// same thread, j = 2..32 in the same warp (shuffles), j = 64, 128 in another
// warp (one shared-memory exchange each).  Padding is +inf (all-ones, INT_MAX).
__global__ void __launch_bounds__(kRunThreads) k_run_sort(const kr_key* keys, const int32_t* idx,
                                                          const unsigned int* count_dev, int m_host,
                                                          kr_key* rk, int32_t* ri) {
    static_assert(kRun == 2 * kRunThreads, "two elements per thread");
    __shared__ Pair sp[kRun];
    const int m = count_dev ? min(static_cast<int>(*count_dev), m_host) : m_host;
    const int base = blockIdx.x * kRun;
    if (base >= m) return;
    const int n = min(kRun, m - base);
    const int t = threadIdx.x;
    Pair e[2];
#pragma unroll
    for (int q = 0; q < 2; q++) {
        const int x = 2 * t + q;
        if (x < n) {
            e[q].k = keys[base + x];
            e[q].i = idx ? idx[base + x] : base + x;
        } else {
            e[q].k = kr_key{~0ull, ~0ull};
            e[q].i = INT_MAX;
        }
    }
#pragma unroll
    for (int kk = 2; kk <= kRun; kk <<= 1) {
        const bool up = ((2 * t) & kk) == 0;  // same for both elements (kk >= 2)
#pragma unroll
        for (int j = kk >> 1; j > 0; j >>= 1) {
            if (j == 1) {
                if (pair_gt(e[0].k, e[0].i, e[1].k, e[1].i) == up) {
                    const Pair tmp = e[0];
                    e[0] = e[1];
                    e[1] = tmp;
                }
            } else {
                const bool lower = ((2 * t) & j) == 0;  // element below its partner
                const bool keep_min = lower == up;
                Pair o[2];
                if (j <= 32) {
                    o[0] = shfl_pair(e[0], j >> 1);
                    o[1] = shfl_pair(e[1], j >> 1);
                } else {
                    sp[2 * t] = e[0];
                    sp[2 * t + 1] = e[1];
                    __syncthreads();
                    o[0] = sp[(2 * t) ^ j];
                    o[1] = sp[(2 * t + 1) ^ j];
                    __syncthreads();
                }
                e[0] = keep(e[0], o[0], keep_min);
                e[1] = keep(e[1], o[1], keep_min);
            }
        }
    }
#pragma unroll
    for (int q = 0; q < 2; q++) {
        const int x = 2 * t + q;
        if (x < n) {
            rk[base + x] = e[q].k;
            ri[base + x] = e[q].i;
        }
    }
}

__device__ __forceinline__ int count_less(const kr_key* rk, const int32_t* ri, int lo, int hi,
                                          const kr_key& x, int32_t xi) {
    const int start = lo;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (pair_gt(x, xi, rk[mid], ri[mid])) lo = mid + 1;
        else hi = mid;
    }
    return lo - start;
}

// One warp per pair: lane r counts the pairs smaller than it in runs
// r, r + 32, ... by binary search (L2-resident), the warp sums the counts and
// lane 0 scatters the pair to its final position.  8 dependent probes per run
// of 256, spread over m warps, keep the whole GPU busy even for small m.
__global__ void __launch_bounds__(256) k_run_merge(const kr_key* rk, const int32_t* ri,
                                                   const unsigned int* count_dev, int m_host,
                                                   int32_t* out_idx, kr_key* out_keys) {
    const int m = count_dev ? min(static_cast<int>(*count_dev), m_host) : m_host;
    const int nruns = (m + kRun - 1) / kRun;
    const int lane = threadIdx.x & 31;
    const int wpb = blockDim.x >> 5;
    for (int e = blockIdx.x * wpb + (threadIdx.x >> 5); e < m; e += gridDim.x * wpb) {
        const kr_key x = rk[e];
        const int32_t xi = ri[e];
        const int own = e / kRun;
        int c = 0;
        for (int r = lane; r < nruns; r += 32)
            if (r != own) c += count_less(rk, ri, r * kRun, min(r * kRun + kRun, m), x, xi);
#pragma unroll
        for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        if (lane == 0) {
            const int rank = c + (e - own * kRun);
            if (out_idx) out_idx[rank] = xi;
            if (out_keys) out_keys[rank] = x;
        }
    }
}

// Small fleets (n <= kSmallAdmit): sort all n (key, index) pairs with the
// run sort (runs of 256 in shared memory on n / 256 CTAs, then the parallel
// rank merge) and apply rank < k as admission (keys are unique, so this is
// key <= kth) -- three short parallel launches instead of the radix select's
// dozen, for latency-bound rounds such as configs[1] (1k robots).
#ifndef KR_SMALL_ADMIT
#define KR_SMALL_ADMIT 16384
#endif
constexpr int kSmallAdmit = KR_SMALL_ADMIT;  // 16k: with the register run sort the
                                             // small path beats the select (configs[2] 91 -> 86 us)

struct SmallAdmitArgs {
    const kr_key* sorted_keys;
    const int32_t* sorted_idx;
    int n, k;
    const int64_t* obs;  // nullable
    int32_t* skipped;    // nullable
    uint8_t* admitted;   // nullable
    uint8_t* refetch;    // nullable
    int64_t now, stale;
    int32_t* edge_idx;   // nullable
    kr_key* edge_keys;   // nullable
    kr_key* kth_out;     // nullable
};

__global__ void __launch_bounds__(256) k_small_apply(SmallAdmitArgs a) {
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < a.n; p += gridDim.x * blockDim.x) {
        const int32_t j = a.sorted_idx[p];
        const bool in = p < a.k;
        if (a.admitted) a.admitted[j] = in;
        if (a.refetch) a.refetch[j] = in && (a.now - __ldg(a.obs + j) > a.stale);
        if (a.skipped) a.skipped[j] = in ? 0 : a.skipped[j] + 1;
        if (in) {
            if (a.edge_idx) a.edge_idx[p] = j;
            if (a.edge_keys) a.edge_keys[p] = a.sorted_keys[p];
        }
        if (a.kth_out && p == a.k - 1) *a.kth_out = a.sorted_keys[p];
    }
}

// Merge of W sorted candidate runs (the sharded round's all-gathered local
// top-k' lists, sentinel-padded to equal length): every element's global rank
// = its index in its run + the number of smaller elements in each other run
// (binary search; one lane per run, a warp per element; ties -- the all-ones
// sentinels -- broken by position).  Ranks < k are the global S_e in order;
// rank k - 1 is the global k-th key.  The protocol is exact only for unique
// keys (global robot ranks, one issued base on every shard): a real key met
// again in another run (or next to itself in its own) sets KR_FLAG_DUP_KEY.
__device__ __forceinline__ bool key_eq(const kr_key& a, const kr_key& b) {
    return a.hi == b.hi && a.lo == b.lo;
}

__global__ void __launch_bounds__(256) k_merge_runs(const kr_key* runs, int W, int len, int k,
                                                    kr_key* out_keys, int32_t* out_pos,
                                                    kr_key* kth_out, uint32_t* flags) {
    const int m = W * len;
    const int lane = threadIdx.x & 31;
    const int wpb = blockDim.x >> 5;
    for (int e = blockIdx.x * wpb + (threadIdx.x >> 5); e < m; e += gridDim.x * wpb) {
        const kr_key x = runs[e];
        const int own = e / len;
        const bool real = ~(x.hi & x.lo) != 0;  // not the all-ones padding
        bool dup = false;
        int c = 0;
        for (int r = lane; r < W; r += 32) {
            int lo = r * len, hi = lo + len;
            const int start = lo, end = hi;
            if (r == own) {
                dup |= real && e > start && key_eq(runs[e - 1], x);
                continue;
            }
            while (lo < hi) {  // elements of run r ordered before (x, e)
                const int mid = (lo + hi) >> 1;
                if (pair_gt(x, e, runs[mid], mid)) lo = mid + 1;
                else hi = mid;
            }
            dup |= real && ((lo > start && key_eq(runs[lo - 1], x)) || (lo < end && key_eq(runs[lo], x)));
            c += lo - start;
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        if (flags && __any_sync(0xffffffffu, dup) && lane == 0) atomicOr(flags, KR_FLAG_DUP_KEY);
        if (lane == 0) {
            const int rank = c + (e - own * len);
            if (rank < k) {
                if (out_keys) out_keys[rank] = x;
                if (out_pos) out_pos[rank] = e;
                if (kth_out && rank == k - 1) *kth_out = x;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// sorting the admitted set (generic paths)
// ---------------------------------------------------------------------------

// --- stable multi-CTA LSD radix sort over 8-bit windows ---------------------
__global__ void __launch_bounds__(256) k_rs_hist(const kr_key* keys, int64_t n, int shift,
                                                 int width, uint32_t* tile_hist, int64_t ntiles) {
    __shared__ unsigned int h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    const int64_t t = blockIdx.x;
    const int64_t lo = t * kSortTile, hi = lo + kSortTile < n ? lo + kSortTile : n;
    const unsigned mask = (1u << width) - 1;
    const int lane = threadIdx.x & 31;
    // warp-aggregated: high windows (bucket, aged estimate) hold few distinct
    // digits, and per-element shared atomics on one bin serialise
    for (int64_t base = lo; base < hi; base += blockDim.x) {
        const int64_t i = base + threadIdx.x;
        unsigned d = 0xFFFFFFFFu;
        if (i < hi) {
            const kr_key k = keys[i];
            d = static_cast<unsigned>(shr128_lo(k.hi, k.lo, shift) & mask);
        }
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        if (d != 0xFFFFFFFFu && lane == __ffs(peers) - 1) atomicAdd(&h[d], __popc(peers));
    }
    __syncthreads();
    tile_hist[static_cast<int64_t>(threadIdx.x) * ntiles + t] = h[threadIdx.x];
}

// Exclusive scan of m entries in place, one CTA of 1024 threads: each thread
// owns a contiguous segment (a multiple of 16 entries), read and rewritten
// with four independent 16-byte accesses per step so the loads overlap.
__global__ void __launch_bounds__(1024) k_rs_scan(uint32_t* a, int64_t m) {
    __shared__ unsigned int part[1024];
    int64_t per = (m + blockDim.x - 1) / blockDim.x;
    per = (per + 15) & ~int64_t(15);
    const int64_t lo = threadIdx.x * per < m ? threadIdx.x * per : m;
    const int64_t hi = lo + per < m ? lo + per : m;
    unsigned int s = 0;
    int64_t i = lo;
    for (; i + 16 <= hi; i += 16) {
        const uint4* q = reinterpret_cast<const uint4*>(a + i);
        const uint4 x0 = q[0], x1 = q[1], x2 = q[2], x3 = q[3];
        s += x0.x + x0.y + x0.z + x0.w + x1.x + x1.y + x1.z + x1.w +
             x2.x + x2.y + x2.z + x2.w + x3.x + x3.y + x3.z + x3.w;
    }
    for (; i < hi; i++) s += a[i];
    part[threadIdx.x] = s;
    __syncthreads();
    for (int o = 1; o < blockDim.x; o <<= 1) {
        unsigned int v = threadIdx.x >= o ? part[threadIdx.x - o] : 0;
        __syncthreads();
        part[threadIdx.x] += v;
        __syncthreads();
    }
    unsigned int run = threadIdx.x ? part[threadIdx.x - 1] : 0;
    i = lo;
    for (; i + 16 <= hi; i += 16) {
        uint4* q = reinterpret_cast<uint4*>(a + i);
        uint4 x[4] = {q[0], q[1], q[2], q[3]};
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const unsigned int v0 = x[j].x, v1 = x[j].y, v2 = x[j].z, v3 = x[j].w;
            x[j].x = run; run += v0;
            x[j].y = run; run += v1;
            x[j].z = run; run += v2;
            x[j].w = run; run += v3;
        }
#pragma unroll
        for (int j = 0; j < 4; j++) q[j] = x[j];
    }
    for (; i < hi; i++) {
        unsigned int v = a[i];
        a[i] = run;
        run += v;
    }
}

__global__ void __launch_bounds__(256) k_rs_scatter(const kr_key* keys, const int32_t* idx,
                                                    int64_t n, int shift, int width,
                                                    const uint32_t* tile_off, int64_t ntiles,
                                                    kr_key* okeys, int32_t* oidx) {
    __shared__ unsigned int wc[8][256];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t t = blockIdx.x;
    const int64_t lo = t * kSortTile;
    const int per_warp = kSortTile / 8;
    const int64_t wlo = lo + warp * per_warp;
    const unsigned mask = (1u << width) - 1;
    for (int d = lane; d < 256; d += 32) wc[warp][d] = 0;
    __syncwarp();
    for (int c = 0; c < per_warp; c += 32) {
        const int64_t i = wlo + c + lane;
        unsigned d = 0xFFFFFFFFu;
        if (i < n) {
            const kr_key k = keys[i];
            d = static_cast<unsigned>(shr128_lo(k.hi, k.lo, shift) & mask);
        }
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        if (d != 0xFFFFFFFFu && lane == __ffs(peers) - 1) wc[warp][d] += __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    {
        unsigned int d = threadIdx.x, run = 0;
        for (int w = 0; w < 8; w++) {
            unsigned int v = wc[w][d];
            wc[w][d] = run;
            run += v;
        }
    }
    __syncthreads();
    for (int c = 0; c < per_warp; c += 32) {
        int64_t i = wlo + c + lane;
        bool valid = i < n;
        kr_key k{0, 0};
        unsigned d = 0xFFFFFFFFu;
        if (valid) {
            k = keys[i];
            d = static_cast<unsigned>(shr128_lo(k.hi, k.lo, shift) & mask);
        }
        unsigned peers = __match_any_sync(0xffffffffu, d);
        unsigned rank = __popc(peers & ((1u << lane) - 1));
        unsigned basew = valid ? wc[warp][d] : 0;
        __syncwarp();
        if (valid) {
            unsigned pos = tile_off[static_cast<int64_t>(d) * ntiles + t] + basew + rank;
            okeys[pos] = k;
            oidx[pos] = idx ? idx[i] : static_cast<int32_t>(i);
            if (rank == 0) wc[warp][d] += __popc(peers);
        }
        __syncwarp();
    }
}

// Sorts (keys, idx) with n elements (keys/idx may alias workspace buffer 0).
static int sort_pairs(const Workspace& w, const kr_key* keys, const int32_t* idx,
                      const unsigned int* count_dev, int64_t n, int32_t* out_idx, kr_key* out_keys,
                      const unsigned long long* stats_dev, cudaStream_t st) {
    if (n <= kRunSortMax) {
        const int m = static_cast<int>(n);
        const kr_key* sk = keys;
        const int32_t* si = idx;
        // runs are written to the sort ping-pong buffer not holding the input
        kr_key* rk = keys == w.skeys[1] ? w.skeys[0] : w.skeys[1];
        int32_t* ri = keys == w.skeys[1] ? w.sidx[0] : w.sidx[1];
        k_run_sort<<<(m + kRun - 1) / kRun, kRunThreads, 0, st>>>(sk, si, count_dev, m, rk, ri);
        const int64_t warps = m;
        int64_t blocks = (warps + 7) / 8;
        if (blocks > 148 * 64) blocks = 148 * 64;
        k_run_merge<<<static_cast<unsigned>(blocks), 256, 0, st>>>(rk, ri, count_dev, m, out_idx,
                                                                   out_keys);
        return check_launch("run sort", 2);
    }
    // window plan from OR ^ AND of the set (read back: one stream sync)
    unsigned long long s4[4];
    KR_CUDA_TRY(cudaMemcpyAsync(s4, stats_dev, sizeof(s4), cudaMemcpyDeviceToHost, st));
    KR_CUDA_TRY(cudaStreamSynchronize(st));
    unsigned long long x[2] = {s4[1] ^ s4[3], s4[0] ^ s4[2]};  // lo, hi
    int shifts[32], widths[32], np = 0;
    for (int b = 0; b < 128;) {
        bool set = (x[b >> 6] >> (b & 63)) & 1ull;
        if (!set) { b++; continue; }
        shifts[np] = b;
        widths[np] = 128 - b < 8 ? 128 - b : 8;
        np++;
        b += 8;
    }
    const int64_t ntiles = static_cast<int64_t>(sort_tiles(n));
    const kr_key* ck = keys;
    const int32_t* ci = idx;
    if (np == 0) {  // all keys identical: one stable pass yields the identity order
        shifts[0] = 0;
        widths[0] = 8;
        np = 1;
    }
    for (int p = 0; p < np; p++) {
        kr_key* ok = w.skeys[p & 1];
        int32_t* oi = w.sidx[p & 1];
        if (ck == ok) { ok = w.skeys[(p + 1) & 1]; oi = w.sidx[(p + 1) & 1]; }
        k_rs_hist<<<static_cast<unsigned>(ntiles), 256, 0, st>>>(ck, n, shifts[p], widths[p],
                                                                 w.tile_hist, ntiles);
        k_rs_scan<<<1, 1024, 0, st>>>(w.tile_hist, ntiles * 256);
        k_rs_scatter<<<static_cast<unsigned>(ntiles), 256, 0, st>>>(
            ck, ci, n, shifts[p], widths[p], w.tile_hist, ntiles, ok, oi);
        int e = check_launch("radix pass", 3);
        if (e) return e;
        ck = ok;
        ci = oi;
    }
    if (out_idx) {
        if (ci)
            KR_CUDA_TRY(cudaMemcpyAsync(out_idx, ci, n * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
        else
            return KR_EINVAL;
    }
    if (out_keys)
        KR_CUDA_TRY(cudaMemcpyAsync(out_keys, ck, n * sizeof(kr_key), cudaMemcpyDeviceToDevice, st));
    return KR_OK;
}

// ---------------------------------------------------------------------------
// Phase 3: hybrid edge / cloud placement (scheduler.py:160-241)
// ---------------------------------------------------------------------------
// engines.py:158-169 transfer_time: base + round_half_up(bytes * 8e6 / bps).
__global__ void k_transfer_time(const int64_t* payload, int64_t n, int64_t base_us, int64_t bps,
                                int64_t* out) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        const unsigned __int128 num = static_cast<unsigned __int128>(payload[i] < 0 ? 0 : payload[i]) * 8000000u;
        const unsigned __int128 den = static_cast<unsigned __int128>(bps);
        out[i] = base_us + static_cast<int64_t>((2 * num + den) / (2 * den));
    }
}

// The reference walks the requests after the edge prefix in order and offloads
// one to the cloud iff  cloud_est(req, c) < edge_est  while c = |S_c| < cap.
// cloud_est = C(c) + up(payload), with C(c) (queue drain + batch latency +
// downlink) non-decreasing in c, so the test is up_r < T(c) = edge_est - C(c),
// T non-increasing (host-computed per round).  With m_r = #{c < cap : T(c) >
// up_r} (a binary search, T being non-increasing) the walk is the recurrence
// fire_r = [c_r < m_r], c_{r+1} = c_r + fire_r.  One CTA takes 1,024 requests
// per window: all threads compute m, then warp 0 resolves the recurrence 32
// requests at a time by a ballot fixed point (lane j fires iff c + fires of
// lanes < j < m_j; iterating from "no earlier fires" fixes at least one more
// lane per round, and the fixed point is the sequential answer), and every
// thread applies its own request's placement.  Accepted requests get their
// skip counter reset and their stale-observation refetch flag
// (scheduler.py:223-234).
__global__ void __launch_bounds__(1024) k_place_cloud(const int32_t* order, int n, int n_edge,
                                                      const int64_t* up, const int64_t* thr,
                                                      int cap, const int64_t* obs, int32_t* skipped,
                                                      uint8_t* refetch, int64_t now, int64_t stale,
                                                      int32_t* cloud_idx, int32_t* n_cloud) {
    __shared__ int s_m[1024];
    __shared__ uint32_t s_fire[32];
    __shared__ int s_pre[32];
    __shared__ int s_c;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_c = 0;
    __syncthreads();
    for (int base = n_edge; base < n; base += 1024) {
        const int c0 = s_c;
        if (c0 >= cap) break;
        const int r = base + tid;
        int m = 0;
        if (r < n) {
            const int64_t u = up[order[r]];
            int lo = 0, hi = cap;  // first c with T(c) <= u
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (thr[mid] > u) lo = mid + 1;
                else hi = mid;
            }
            m = lo;
        }
        s_m[tid] = m;
        __syncthreads();
        if (warp == 0) {
            int cc = c0;
            const uint32_t below = (1u << lane) - 1u;
            for (int ch = 0; ch < 32; ch++) {
                const int mm = s_m[ch * 32 + lane];
                uint32_t f = __ballot_sync(0xffffffffu, cc < mm);
                for (;;) {
                    const uint32_t g = __ballot_sync(0xffffffffu, cc + __popc(f & below) < mm);
                    if (g == f) break;
                    f = g;
                }
                if (lane == 0) {
                    s_fire[ch] = f;
                    s_pre[ch] = cc;
                }
                cc += __popc(f);
            }
            if (lane == 0) s_c = cc;
        }
        __syncthreads();
        const uint32_t f = s_fire[warp];
        if ((f >> lane) & 1u) {
            const int slot = s_pre[warp] + __popc(f & ((1u << lane) - 1u));
            const int i = order[r];
            cloud_idx[slot] = i;
            if (skipped) skipped[i] = 0;
            if (refetch) refetch[i] = now - obs[i] > stale;
        }
        __syncthreads();
    }
    if (tid == 0) *n_cloud = s_c;
}

static unsigned grid_stream(int64_t n) {
    int64_t b = (n + 255) / 256;
    int64_t cap = static_cast<int64_t>(device_info().sm_count) * 8;
    if (b > cap) b = cap;
    return static_cast<unsigned>(b < 1 ? 1 : b);
}

}  // namespace kr

using namespace kr;

extern "C" size_t kr_workspace_bytes(int64_t n) { return workspace_bytes(n); }

// Launches the select pipeline (workspace state left holding the level-0
// k-th key in state->kth).  Returns KR_OK or an error.
static int select_pipeline(const kr_key* keys, int64_t n, int64_t k,
                           const unsigned long long* key_stats, const Workspace& w,
                           cudaStream_t st) {
    SelState* s = w.state;
    k_sel_reset<<<1, 1024, 0, st>>>(s, n, k, key_stats);
    int launches = 1;
    if (!key_stats) {
        k_sel_stats<<<grid_stream(n), 256, 0, st>>>(keys, n, s);
        launches++;
    }
    // level 0: all keys -> cand[0]; level 1: cand[0] -> cand[1]; finisher reads cand[1]
    k_sel_hist<<<grid_stream(n), 256, 0, st>>>(keys, s, 0);
    k_sel_pick<<<1, 1024, 0, st>>>(s, keys, 0);
    k_sel_scatter<<<grid_stream(n), 256, 0, st>>>(keys, w.cand[0], s, 0);
    k_sel_hist<<<grid_stream(n / 64 + 1), 256, 0, st>>>(w.cand[0], s, 1);
    k_sel_pick<<<1, 1024, 0, st>>>(s, w.cand[0], 1);
    k_sel_scatter<<<grid_stream(n / 64 + 1), 256, 0, st>>>(w.cand[0], w.cand[1], s, 1);
    k_sel_finish<<<1, 1024, 0, st>>>(s, w.cand[1], w.cand[0], 2);
    return check_launch("select", launches + 7);
}

static int admit_with(const kr_key* keys, int64_t n, int64_t k, const kr_key* kth,
                      const kr_fleet* fleet, const kr_sched* cfg, uint8_t* admitted,
                      uint8_t* refetch, int32_t* edge_idx, kr_key* edge_keys, const Workspace& w,
                      cudaStream_t st);

extern "C" int kr_key_stats_init(unsigned long long* stats, void* stream) {
    if (!stats) return KR_EINVAL;
    cudaStream_t st = as_stream(stream);
    KR_CUDA_TRY(cudaMemsetAsync(stats, 0, 2 * sizeof(unsigned long long), st));
    KR_CUDA_TRY(cudaMemsetAsync(stats + 2, 0xFF, 2 * sizeof(unsigned long long), st));
    return KR_OK;
}

extern "C" int kr_select_admit(const kr_key* keys, int64_t n, int64_t k,
                               const unsigned long long* key_stats, const kr_fleet* fleet,
                               const kr_sched* cfg, uint8_t* admitted, uint8_t* refetch,
                               int32_t* edge_idx, kr_key* edge_keys, kr_key* kth_out, void* ws,
                               size_t ws_bytes, void* stream);

extern "C" int kr_merge_runs_pos(const kr_key* runs, int32_t W, int64_t len, int64_t k,
                                 kr_key* out_keys, int32_t* out_pos, kr_key* kth_out,
                                 uint32_t* flags, void* stream) {
    if (W < 1 || len < 0 || k < 0 || k > static_cast<int64_t>(W) * len ||
        static_cast<int64_t>(W) * len > INT_MAX)
        return KR_EINVAL;
    if (k == 0 || len == 0) return KR_OK;
    if (!runs) return KR_EINVAL;
    const int64_t m = static_cast<int64_t>(W) * len;
    int64_t blocks = (m + 7) / 8;
    const int64_t cap = static_cast<int64_t>(device_info().sm_count) * 64;
    if (blocks > cap) blocks = cap;
    k_merge_runs<<<static_cast<unsigned>(blocks), 256, 0, as_stream(stream)>>>(
        runs, W, static_cast<int>(len), static_cast<int>(k), out_keys, out_pos, kth_out, flags);
    return check_launch("kr_merge_runs");
}

extern "C" int kr_merge_runs(const kr_key* runs, int32_t W, int64_t len, int64_t k,
                             kr_key* out_keys, kr_key* kth_out, uint32_t* flags, void* stream) {
    return kr_merge_runs_pos(runs, W, len, k, out_keys, nullptr, kth_out, flags, stream);
}

extern "C" int kr_topk_select(const kr_key* keys, int64_t n, int64_t k, kr_key* kth,
                              const unsigned long long* key_stats, void* ws, size_t ws_bytes,
                              void* stream) {
    if (n < 0 || k < 0 || !kth) return KR_EINVAL;
    cudaStream_t st = as_stream(stream);
    if (k == 0 || n == 0) return KR_OK;
    if (k >= n) {
        k_set_key<<<1, 1, 0, st>>>(kth, ~0ull, ~0ull);
        return check_launch("kr_topk_select");
    }
    if (!ws || ws_bytes < workspace_bytes(n) || !keys) return KR_ENOSPACE;
    Workspace w = carve(ws, n);
    int e = select_pipeline(keys, n, k, key_stats, w, st);
    if (e) return e;
    k_copy_kth<<<1, 1, 0, st>>>(w.state, kth);
    return check_launch("kr_topk_select");
}

extern "C" int kr_select_admit(const kr_key* keys, int64_t n, int64_t k,
                               const unsigned long long* key_stats, const kr_fleet* fleet,
                               const kr_sched* cfg, uint8_t* admitted, uint8_t* refetch,
                               int32_t* edge_idx, kr_key* edge_keys, kr_key* kth_out, void* ws,
                               size_t ws_bytes, void* stream) {
    if (n < 0 || k < 0) return KR_EINVAL;
    if (n == 0) return KR_OK;
    if (!keys) return KR_EINVAL;
    if ((refetch || (fleet && fleet->skipped)) && (!fleet || !cfg)) return KR_EINVAL;
    if (!ws || ws_bytes < workspace_bytes(n)) return KR_ENOSPACE;
    cudaStream_t st = as_stream(stream);
    if (k == 0 || k >= n) {  // nothing to select: generic admission (+ full order if k >= n)
        const kr_key* kth_ptr = nullptr;
        if (kth_out && k >= n) {
            k_set_key<<<1, 1, 0, st>>>(kth_out, ~0ull, ~0ull);
            int e = check_launch("kr_select_admit");
            if (e) return e;
        }
        return kr_admit(keys, n, k, kth_ptr, fleet, cfg, admitted, refetch, edge_idx, edge_keys,
                        ws, ws_bytes, stream);
    }
    if (n <= kSmallAdmit) {  // sort everything (run sort), rank < k is admission
        Workspace w = carve(ws, n);
        int e = sort_pairs(w, keys, nullptr, nullptr, n, w.sidx[0], w.skeys[0], nullptr, st);
        if (e) return e;
        SmallAdmitArgs a{};
        a.sorted_keys = w.skeys[0];
        a.sorted_idx = w.sidx[0];
        a.n = static_cast<int>(n);
        a.k = static_cast<int>(k);
        a.obs = fleet ? fleet->obs_captured_at : nullptr;
        a.skipped = fleet ? fleet->skipped : nullptr;
        a.admitted = admitted;
        a.refetch = refetch;
        a.now = cfg ? cfg->now : 0;
        a.stale = cfg ? cfg->stale_threshold : 0;
        a.edge_idx = edge_idx;
        a.edge_keys = edge_keys;
        a.kth_out = kth_out;
        k_small_apply<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(a);
        return check_launch("kr_select_admit(small)");
    }
    Workspace w = carve(ws, n);
    int e = select_pipeline(keys, n, k, key_stats, w, st);
    if (e) return e;
    if (kth_out) {
        k_copy_kth<<<1, 1, 0, st>>>(w.state, kth_out);
        e = check_launch("kr_select_admit");
        if (e) return e;
    }
    return admit_with(keys, n, k, &w.state->kth, fleet, cfg, admitted, refetch, edge_idx,
                      edge_keys, w, st);
}

// Admission pass + (optional) ordered gather of the admitted set.
static int admit_with(const kr_key* keys, int64_t n, int64_t k, const kr_key* kth,
                      const kr_fleet* fleet, const kr_sched* cfg, uint8_t* admitted,
                      uint8_t* refetch, int32_t* edge_idx, kr_key* edge_keys, const Workspace& w,
                      cudaStream_t st) {
    const bool gather = edge_idx || edge_keys;
    if (gather) k_admit_init<<<1, 32, 0, st>>>(w.state);
    AdmitArgs a{};
    a.keys = keys;
    a.n = n;
    a.all = kth == nullptr;
    a.none = k == 0;
    a.kth = kth;
    a.obs = fleet ? fleet->obs_captured_at : nullptr;
    a.skipped = fleet ? fleet->skipped : nullptr;
    a.admitted = admitted;
    a.refetch = refetch;
    a.now = cfg ? cfg->now : 0;
    a.stale = cfg ? cfg->stale_threshold : 0;
    a.sel_keys = gather ? w.skeys[0] : nullptr;
    a.sel_idx = gather ? w.sidx[0] : nullptr;
    a.s = w.state;
    k_admit<<<grid_stream(n), 256, 0, st>>>(a);
    int e = check_launch("k_admit", gather ? 2 : 1);
    if (e || !gather) return e;
    const int64_t m = k < n ? k : n;
    if (m == 0) return KR_OK;
    return sort_pairs(w, w.skeys[0], w.sidx[0], m <= kRunSortMax ? &w.state->sel_count : nullptr,
                      m, edge_idx, edge_keys, w.state->sst, st);
}

extern "C" int kr_admit(const kr_key* keys, int64_t n, int64_t k, const kr_key* kth,
                        const kr_fleet* fleet, const kr_sched* cfg, uint8_t* admitted,
                        uint8_t* refetch, int32_t* edge_idx, kr_key* edge_keys, void* ws,
                        size_t ws_bytes, void* stream) {
    if (n < 0 || k < 0) return KR_EINVAL;
    if (n == 0) return KR_OK;
    if (!keys) return KR_EINVAL;
    if ((refetch || (fleet && fleet->skipped)) && (!fleet || !cfg)) return KR_EINVAL;
    const bool gather = edge_idx || edge_keys;
    Workspace w{};
    if (gather) {
        if (!ws || ws_bytes < workspace_bytes(n)) return KR_ENOSPACE;
        w = carve(ws, n);
    }
    return admit_with(keys, n, k, kth, fleet, cfg, admitted, refetch, edge_idx, edge_keys, w,
                      as_stream(stream));
}

extern "C" int kr_sort_keys(const kr_key* keys, int64_t n, int32_t* order, kr_key* sorted_keys,
                            void* ws, size_t ws_bytes, void* stream) {
    if (n < 0) return KR_EINVAL;
    if (n == 0) return KR_OK;
    if (!keys || !ws || ws_bytes < workspace_bytes(n)) return KR_ENOSPACE;
    cudaStream_t st = as_stream(stream);
    Workspace w = carve(ws, n);
    if (n <= kRunSortMax)
        return sort_pairs(w, keys, nullptr, nullptr, n, order, sorted_keys, nullptr, st);
    k_sel_reset<<<1, 1024, 0, st>>>(w.state, n, 0, nullptr);
    k_sel_stats<<<grid_stream(n), 256, 0, st>>>(keys, n, w.state);
    int e = check_launch("kr_sort_keys", 2);
    if (e) return e;
    return sort_pairs(w, keys, nullptr, nullptr, n, order, sorted_keys, w.state->st[0], st);
}

extern "C" int kr_transfer_time(const int64_t* payload, int64_t n, int64_t base_us, int64_t bps,
                                int64_t* out, void* stream) {
    if (n < 0 || bps <= 0) return KR_EINVAL;
    if (n == 0) return KR_OK;
    if (!payload || !out) return KR_EINVAL;
    k_transfer_time<<<grid_stream(n), 256, 0, as_stream(stream)>>>(payload, n, base_us, bps, out);
    return check_launch("kr_transfer_time");
}

extern "C" int kr_place_cloud(const int32_t* order, int64_t n, int64_t n_edge,
                              const int64_t* up_us, const int64_t* thresholds, int64_t cap,
                              const kr_fleet* fleet, const kr_sched* cfg, uint8_t* refetch,
                              int32_t* cloud_idx, int32_t* n_cloud, void* stream) {
    if (n < 0 || n_edge < 0 || cap < 0 || n > INT32_MAX) return KR_EINVAL;
    if (!n_cloud) return KR_EINVAL;
    cudaStream_t st = as_stream(stream);
    if (n == 0 || cap == 0 || n_edge >= n) {
        KR_CUDA_TRY(cudaMemsetAsync(n_cloud, 0, sizeof(int32_t), st));
        return KR_OK;
    }
    if (!order || !up_us || !thresholds || !cloud_idx) return KR_EINVAL;
    if (refetch && (!fleet || !cfg)) return KR_EINVAL;
    k_place_cloud<<<1, 1024, 0, st>>>(order, static_cast<int>(n), static_cast<int>(n_edge), up_us,
                                      thresholds, static_cast<int>(cap),
                                      fleet ? fleet->obs_captured_at : nullptr,
                                      fleet ? fleet->skipped : nullptr, refetch,
                                      cfg ? cfg->now : 0, cfg ? cfg->stale_threshold : 0,
                                      cloud_idx, n_cloud);
    return check_launch("kr_place_cloud");
}
