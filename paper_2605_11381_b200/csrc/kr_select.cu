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
#include "kr_select_state.cuh"

namespace kr {

#ifndef KR_SEL_U
#define KR_SEL_U 4
#endif
constexpr int kSelU = KR_SEL_U;  // keys in flight per thread in the level-0 histogram
#ifndef KR_SCAT_W
#define KR_SCAT_W 1
#endif
constexpr int kScatW = KR_SCAT_W;  // digits per thread per step in the level-0 scatter
#ifndef KR_SORT_TILE
#define KR_SORT_TILE 4096
#endif
constexpr int kSortTile = KR_SORT_TILE;  // LSD radix: elements per CTA tile (256 threads x 16)

struct Workspace {
    SelState* state;
    uint16_t* digits;  // level-0 digit of every key
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
    b += align256(nn * sizeof(uint16_t));        // level-0 digits
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
    w.digits = reinterpret_cast<uint16_t*>(p);
    p += align256(nn * sizeof(uint16_t));
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
// Three launches: k_sel_reset (state, level-0 digit from the keys' OR / AND),
// k_sel_hist0 (every key's digit -> a 16-bit digit array + the histogram; the
// last CTA to finish picks the boundary bin d*) and k_sel_scatter0 (the keys
// of bin d*, read through the digit array, -> candidates; the last CTA runs
// the remaining levels over the candidates alone and publishes the k-th key).
// The admission pass then decides most keys from the digit array alone
// (digit < d*: in, > d*: out).  "Last CTA" = the CTA whose increment of a
// completion counter returns gridDim - 1, after a release fence by every CTA.

__global__ void k_sel_reset(SelState* s, int64_t n, int64_t k, const unsigned long long* stats,
                            const kr_key* keys) {
    for (int i = threadIdx.x; i < kBins; i += blockDim.x) s->hist[i] = 0;
    if (threadIdx.x == 0) {
        s->st[0][0] = 0; s->st[0][1] = 0; s->st[0][2] = ~0ull; s->st[0][3] = ~0ull;
        sel_init(s, n, k);
        if (stats) {
            for (int j = 0; j < 4; j++) s->st[0][j] = stats[j];
            sel_digit0(s, keys);
        }
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
__global__ void k_sel_digit(SelState* s, const kr_key* keys) { sel_digit0(s, keys); }

// True in every thread of the CTA that completes the grid pass last.
__device__ __forceinline__ bool last_cta(unsigned int* counter) {
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(counter, 1u) == gridDim.x - 1;
    __syncthreads();
    if (last) __threadfence();
    return last;
}

// One block: choose the boundary bin d* (cum_lt < need <= cum_le) of `hist`
// (bins of digit d; shared memory or this CTA's own data).
__device__ void sel_pick_block(SelState* s, const Digit& d, const unsigned int* hist) {
    __shared__ unsigned int part[1024];
    const int bins = 1 << d.W;
    const int nt = blockDim.x;
    const int per = (bins + nt - 1) / nt;
    unsigned int local = 0;
    for (int q = 0; q < per; q++) {
        int b = threadIdx.x * per + q;
        if (b < bins) local += hist[b];
    }
    part[threadIdx.x] = local;
    __syncthreads();
    // inclusive scan of part[] (Hillis-Steele)
    for (int o = 1; o < nt; o <<= 1) {
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
                break;
            }
            cum += c;
        }
    }
    __syncthreads();
}

// Level 0 over all keys: digits[i] and the histogram; the last CTA picks d*.
__global__ void __launch_bounds__(256) k_sel_hist0(const kr_key* __restrict__ keys, int64_t n,
                                                   uint16_t* __restrict__ digits, SelState* s) {
    griddep_wait();
    __shared__ unsigned int h[kBins];
    __shared__ Digit sd;
    __shared__ int sdone;
    if (threadIdx.x == 0) {
        sd = s->d0;
        sdone = s->done;
    }
    for (int i = threadIdx.x; i < kBins; i += blockDim.x) h[i] = 0;
    __syncthreads();
    const Digit d = sd;
    if (!sdone) {
        // kSelU keys in flight per thread
        const int64_t T = blockDim.x;
        for (int64_t base = blockIdx.x * T * kSelU; base < n; base += int64_t(gridDim.x) * T * kSelU) {
            kr_key kk[kSelU];
#pragma unroll
            for (int u = 0; u < kSelU; u++) {
                const int64_t i = base + u * T + threadIdx.x;
                if (i < n) kk[u] = keys[i];
            }
#pragma unroll
            for (int u = 0; u < kSelU; u++) {
                const int64_t i = base + u * T + threadIdx.x;
                if (i < n) {
                    const unsigned v = digit_val(kk[u], d);
                    digits[i] = static_cast<uint16_t>(v);
                    atomicAdd(&h[v], 1u);
                }
            }
        }
        __syncthreads();
        const int bins = 1 << d.W;
        for (int i = threadIdx.x; i < bins; i += blockDim.x)
            if (h[i]) atomicAdd(&s->hist[i], h[i]);
    }
    if (!last_cta(&s->done_hist) || sdone) return;
    const int bins = 1 << d.W;
    for (int i = threadIdx.x; i < bins; i += blockDim.x) h[i] = __ldcg(&s->hist[i]);
    __syncthreads();
    sel_pick_block(s, d, h);
    if (threadIdx.x == 0) s->dstar0 = s->dstar;
}

// Remaining levels over the candidates (count cnt[p], OR / AND st[p]) in one
// CTA, ping-ponging between src and dst, until one key remains.
__device__ void sel_finish_block(SelState* s, kr_key* src, kr_key* dst, int p) {
    __shared__ unsigned int h[kBins];
    __shared__ unsigned long long sst[4];
    __shared__ unsigned int scnt;
    __shared__ unsigned int sn, sdstar, ssingle;
    __shared__ unsigned long long stin[4];
    for (int it = 0; it < 130; it++) {
        // L2 reads: the first level's count and OR / AND come from other CTAs
        if (threadIdx.x == 0) sn = __ldcg(&s->cnt[p]);
        if (threadIdx.x < 4) stin[threadIdx.x] = __ldcg(&s->st[p][threadIdx.x]);
        __syncthreads();
        const unsigned n = sn;
        const Digit d = digit_of(stin);
        if (!d.any || n <= 1) {
            if (threadIdx.x == 0) {
                s->kth = src[0];
                s->done = 1;
            }
            __syncthreads();
            return;
        }
        const int bins = 1 << d.W;
        for (int i = threadIdx.x; i < bins; i += blockDim.x) h[i] = 0;
        __syncthreads();
        for (unsigned i = threadIdx.x; i < n; i += blockDim.x) atomicAdd(&h[digit_val(src[i], d)], 1u);
        __syncthreads();
        sel_pick_block(s, d, h);
        if (threadIdx.x == 0) {
            sdstar = s->dstar;
            ssingle = s->dcount == 1;
        }
        if (threadIdx.x < 4) sst[threadIdx.x] = threadIdx.x < 2 ? 0ull : ~0ull;
        if (threadIdx.x == 0) scnt = 0;
        __syncthreads();
        const unsigned dstar = sdstar;
        const bool single = ssingle;
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
        if (single) {
            __syncthreads();
            return;
        }
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

// The keys of bin d* -> cand (through the digit array; single-key bin: the
// answer), then in the last CTA the remaining levels; kth_out (nullable)
// receives the k-th key.
__global__ void __launch_bounds__(256) k_sel_scatter0(const kr_key* __restrict__ keys, int64_t n,
                                                      const uint16_t* __restrict__ digits,
                                                      kr_key* cand, kr_key* spare, SelState* s,
                                                      kr_key* kth_out) {
    griddep_wait();
    __shared__ unsigned sdstar;
    __shared__ int ssingle, sdone;
    if (threadIdx.x == 0) {
        sdstar = s->dstar;
        ssingle = s->dcount == 1;
        sdone = s->done;
    }
    __syncthreads();
    const unsigned dstar = sdstar;
    const bool single = ssingle;
    unsigned long long oh = 0, ol = 0, ah = ~0ull, al = ~0ull;
    if (!sdone) {
        // kScatW digits per thread per step (8: one 16-byte load)
        const int lane = threadIdx.x & 31;
        const int64_t stride = int64_t(gridDim.x) * blockDim.x * kScatW;
        for (int64_t base = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) * kScatW;
             base - threadIdx.x * kScatW < n; base += stride) {
            uint16_t dg[kScatW];
            if (kScatW == 8 && base + 8 <= n) {
                const uint4 v = *reinterpret_cast<const uint4*>(digits + base);
                const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int u = 0; u < kScatW; u++)
                    dg[u] = static_cast<uint16_t>(w[(u >> 1) & 3] >> (16 * (u & 1)));
            } else {
#pragma unroll
                for (int u = 0; u < kScatW; u++) dg[u] = base + u < n ? digits[base + u] : 0xFFFFu;
            }
#pragma unroll
            for (int u = 0; u < kScatW; u++) {
                const bool keep = dg[u] == dstar && base + u < n;
                kr_key k{0, 0};
                if (keep) k = keys[base + u];
                if (single) {
                    if (keep) {
                        s->kth = k;
                        s->done = 1;
                    }
                    continue;
                }
                const unsigned mask = __ballot_sync(0xffffffffu, keep);
                if (mask) {
                    const int leader = __ffs(mask) - 1;
                    unsigned bp = 0;
                    if (lane == leader) bp = atomicAdd(&s->cnt[1], __popc(mask));
                    bp = __shfl_sync(0xffffffffu, bp, leader);
                    if (keep) {
                        cand[bp + __popc(mask & ((1u << lane) - 1))] = k;
                        oh |= k.hi; ol |= k.lo; ah &= k.hi; al &= k.lo;
                    }
                }
            }
        }
        if (!single) stats_accumulate(s->st[1], oh, ol, ah, al);
    }
    if (!last_cta(&s->done_scatter)) return;
    if (!__ldcg(&s->done)) sel_finish_block(s, cand, spare, 1);
    if (kth_out && threadIdx.x == 0) {
        const ulonglong2 v = __ldcg(reinterpret_cast<const ulonglong2*>(&s->kth));
        *kth_out = kr_key{v.x, v.y};
    }
}

__global__ void k_set_key(kr_key* dst, unsigned long long hi, unsigned long long lo) {
    dst->hi = hi;
    dst->lo = lo;
}

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
    const uint16_t* digits; // nullable: level-0 digits of the select that produced kth
};

__global__ void k_admit_init(SelState* s) {
    if (threadIdx.x == 0) {
        s->sel_count = 0;
        s->sst[0] = 0; s->sst[1] = 0; s->sst[2] = ~0ull; s->sst[3] = ~0ull;
    }
}

// One thread per request.  After the fused select the digit array decides a
// request without its key unless its digit is the boundary bin's.  Admitted
// (key, index) pairs are appended per warp (one atomic per warp; their order
// is fixed by the sort that follows).
__global__ void __launch_bounds__(256) k_admit(AdmitArgs a) {
    griddep_wait();
    kr_key kth{~0ull, ~0ull};
    if (!a.all && !a.none) kth = *a.kth;
    const bool dig = a.digits && !a.all && !a.none;
    const unsigned dstar = dig ? a.s->dstar0 : 0u;
    unsigned long long oh = 0, ol = 0, ah = ~0ull, al = ~0ull;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    const int lane = threadIdx.x & 31;
    for (int64_t base = blockIdx.x * int64_t(blockDim.x); base < a.n; base += stride) {
        int64_t i = base + threadIdx.x;
        bool in = false;
        kr_key k{0, 0};
        if (i < a.n) {
            if (dig) {  // after the fused select: the digit decides outside bin d*
                const unsigned dg = a.digits[i];
                if (dg == dstar) {
                    k = a.keys[i];
                    in = key_le(k, kth);
                } else {
                    in = dg < dstar;
                    if (in && a.sel_keys) k = a.keys[i];
                }
            } else {
                k = a.keys[i];
                in = !a.none && (a.all || key_le(k, kth));
            }
            if (a.admitted) a.admitted[i] = in;
            if (a.refetch) a.refetch[i] = in && (a.now - __ldg(a.obs + i) > a.stale);
            if (a.skipped) a.skipped[i] = in ? 0 : a.skipped[i] + 1;
        }
        if (a.sel_keys) {
            const unsigned mask = __ballot_sync(0xffffffffu, in);
            if (mask) {
                const int leader = __ffs(mask) - 1;
                unsigned bp = 0;
                if (lane == leader) bp = atomicAdd(&a.s->sel_count, __popc(mask));
                bp = __shfl_sync(0xffffffffu, bp, leader);
                if (in) {
                    const unsigned pos = bp + __popc(mask & ((1u << lane) - 1));
                    a.sel_keys[pos] = k;
                    a.sel_idx[pos] = static_cast<int32_t>(i);
                    oh |= k.hi; ol |= k.lo; ah &= k.hi; al &= k.lo;
                }
            }
        }
    }
    if (a.sel_keys) stats_accumulate(a.s->sst, oh, ol, ah, al);
}

// The admission pass after the fused select: four requests per thread with
// vector loads / stores of the digit, skip-counter, admitted and refetch
// columns; a request's key is read only in the boundary bin (or, when
// gathering, if admitted), its observation time only if admitted.
__global__ void __launch_bounds__(256) k_admit_dig(AdmitArgs a) {
    const kr_key kth = *a.kth;
    const unsigned dstar = a.s->dstar0;
    const int lane = threadIdx.x & 31;
    unsigned long long oh = 0, ol = 0, ah = ~0ull, al = ~0ull;
    const int64_t n = a.n;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x * 4;
    for (int64_t base = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) * 4;
         base - threadIdx.x * 4 < n; base += stride) {
        const bool full = base + 4 <= n;
        unsigned dg[4];
        int32_t sk[4] = {0, 0, 0, 0};
        if (full) {
            const uint2 v = *reinterpret_cast<const uint2*>(a.digits + base);
            dg[0] = v.x & 0xFFFFu; dg[1] = v.x >> 16; dg[2] = v.y & 0xFFFFu; dg[3] = v.y >> 16;
            if (a.skipped) {
                const int4 q = *reinterpret_cast<const int4*>(a.skipped + base);
                sk[0] = q.x; sk[1] = q.y; sk[2] = q.z; sk[3] = q.w;
            }
        } else {
#pragma unroll
            for (int u = 0; u < 4; u++) {
                dg[u] = base + u < n ? a.digits[base + u] : 0xFFFFFFFFu;
                if (a.skipped && base + u < n) sk[u] = a.skipped[base + u];
            }
        }
        bool in[4];
        kr_key kk[4];
#pragma unroll
        for (int u = 0; u < 4; u++) {
            in[u] = false;
            kk[u] = kr_key{0, 0};
            if (base + u < n) {
                if (dg[u] == dstar) {
                    kk[u] = a.keys[base + u];
                    in[u] = key_le(kk[u], kth);
                } else {
                    in[u] = dg[u] < dstar;
                    if (in[u] && a.sel_keys) kk[u] = a.keys[base + u];
                }
            }
        }
        uint32_t adm = 0, ref = 0;
#pragma unroll
        for (int u = 0; u < 4; u++) {
            adm |= static_cast<uint32_t>(in[u]) << (8 * u);
            if (a.refetch && in[u] && a.now - __ldg(a.obs + base + u) > a.stale) ref |= 1u << (8 * u);
            sk[u] = in[u] ? 0 : sk[u] + 1;
        }
        if (full) {
            if (a.admitted) *reinterpret_cast<uint32_t*>(a.admitted + base) = adm;
            if (a.refetch) *reinterpret_cast<uint32_t*>(a.refetch + base) = ref;
            if (a.skipped) *reinterpret_cast<int4*>(a.skipped + base) = make_int4(sk[0], sk[1], sk[2], sk[3]);
        } else {
#pragma unroll
            for (int u = 0; u < 4; u++) {
                if (base + u >= n) break;
                if (a.admitted) a.admitted[base + u] = static_cast<uint8_t>((adm >> (8 * u)) & 1u);
                if (a.refetch) a.refetch[base + u] = static_cast<uint8_t>((ref >> (8 * u)) & 1u);
                if (a.skipped) a.skipped[base + u] = sk[u];
            }
        }
        if (a.sel_keys) {
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const unsigned mask = __ballot_sync(0xffffffffu, in[u]);
                if (!mask) continue;
                const int leader = __ffs(mask) - 1;
                unsigned bp = 0;
                if (lane == leader) bp = atomicAdd(&a.s->sel_count, __popc(mask));
                bp = __shfl_sync(0xffffffffu, bp, leader);
                if (in[u]) {
                    const unsigned pos = bp + __popc(mask & ((1u << lane) - 1));
                    a.sel_keys[pos] = kk[u];
                    a.sel_idx[pos] = static_cast<int32_t>(base + u);
                    oh |= kk[u].hi; ol |= kk[u].lo; ah &= kk[u].hi; al &= kk[u].lo;
                }
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

// The admission writes of the small-fleet path for the pair at plan position
// p (request j, key x): rank < k is admission (keys are unique), refetch of a
// stale observation, skip counter, ordered S_e and the k-th key.
__device__ __forceinline__ void apply_one(const SmallAdmitArgs& a, int p, int32_t j, const kr_key& x) {
    const bool in = p < a.k;
    if (a.admitted) a.admitted[j] = in;
    if (a.refetch) a.refetch[j] = in && (a.now - __ldg(a.obs + j) > a.stale);
    if (a.skipped) a.skipped[j] = in ? 0 : a.skipped[j] + 1;
    if (in) {
        if (a.edge_idx) a.edge_idx[p] = j;
        if (a.edge_keys) a.edge_keys[p] = x;
    }
    if (a.kth_out && p == a.k - 1) *a.kth_out = x;
}

// One run of kRun = 256 pairs per CTA, a bitonic network held in registers:
// thread t owns elements 2t and 2t + 1; partners at distance j = 1 are in the
// same thread, j = 2..32 in the same warp (shuffles), j = 64, 128 in another
// warp (one shared-memory exchange each).  Padding is +inf (all-ones, INT_MAX).
__global__ void __launch_bounds__(kRunThreads) k_run_sort(const kr_key* keys, const int32_t* idx,
                                                          const unsigned int* count_dev, int m_host,
                                                          kr_key* rk, int32_t* ri,
                                                          SmallAdmitArgs a = SmallAdmitArgs{},
                                                          int apply = 0) {
    griddep_wait();
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
            if (apply) {  // a single run is the whole order: admission from the registers
                apply_one(a, base + x, e[q].i, e[q].k);
            } else {
                rk[base + x] = e[q].k;
                ri[base + x] = e[q].i;
            }
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
                                                   int32_t* out_idx, kr_key* out_keys,
                                                   SmallAdmitArgs a = SmallAdmitArgs{}, int apply = 0) {
    griddep_wait();
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
            if (apply) {
                apply_one(a, rank, xi, x);
            } else {
                if (out_idx) out_idx[rank] = xi;
                if (out_keys) out_keys[rank] = x;
            }
        }
    }
}

// Grouped rank merge: sorted runs of length L, merged G at a time (G a power
// of two <= 32): a sub-warp of G lanes per pair, lane j counting the pairs
// smaller than it in run j of the pair's group (one binary search of log2 L
// dependent probes), the sub-warp sums, lane 0 scatters the pair to its rank
// inside the group's output segment.  Repeated passes (G = 8 until at most 8
// runs remain) replace one pass against every other run: at 16k pairs
// (64 runs) 2 passes of 7 searches instead of 63 searches per pair.
__global__ void __launch_bounds__(256) k_run_merge_group(const kr_key* rk, const int32_t* ri,
                                                         const unsigned int* count_dev, int m_host,
                                                         int L, int lgG, int32_t* out_idx,
                                                         kr_key* out_keys,
                                                         SmallAdmitArgs a = SmallAdmitArgs{},
                                                         int apply = 0) {
    griddep_wait();
    const int m = count_dev ? min(static_cast<int>(*count_dev), m_host) : m_host;
    const int G = 1 << lgG;
    const int nruns = (m + L - 1) / L;
    const int lane = threadIdx.x & 31;
    const int gl = lane & (G - 1);
    const int spw = 32 >> lgG;  // pairs per warp
    const int64_t warp = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
    const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t e0 = warp * spw; e0 < m; e0 += nwarps * spw) {  // warp-uniform
        const int e = static_cast<int>(e0) + (lane >> lgG);
        const bool ok = e < m;
        kr_key x{0, 0};
        int32_t xi = 0;
        int run = 0, c = 0;
        if (ok) {
            x = rk[e];
            xi = ri[e];
            run = e / L;
            const int r = (run & ~(G - 1)) + gl;
            if (r != run && r < nruns) c = count_less(rk, ri, r * L, min(r * L + L, m), x, xi);
        }
        for (int o = G >> 1; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        if (ok && gl == 0) {
            const int pos = (run & ~(G - 1)) * L + c + (e - run * L);
            if (apply) {
                apply_one(a, pos, xi, x);
            } else {
                if (out_idx) out_idx[pos] = xi;
                if (out_keys) out_keys[pos] = x;
            }
        }
    }
}

// The same rank merge with every 16th pair of every run staged in shared
// memory (m <= kMergeSampled): a lane finds its run's 16-pair window among the
// samples, then counts inside the window with 15 independent loads -- one
// L2 latency per lane instead of eight dependent probes.
constexpr int kMergeStep = 16;
constexpr int kMergeSampled = 16384;
__global__ void __launch_bounds__(256) k_run_merge_sampled(const kr_key* rk, const int32_t* ri,
                                                           const unsigned int* count_dev, int m_host,
                                                           int32_t* out_idx, kr_key* out_keys) {
    __shared__ kr_key sk[kMergeSampled / kMergeStep];
    __shared__ int32_t si[kMergeSampled / kMergeStep];
    const int m = count_dev ? min(static_cast<int>(*count_dev), m_host) : m_host;
    const int ns = (m + kMergeStep - 1) / kMergeStep;
    for (int j = threadIdx.x; j < ns; j += blockDim.x) {
        sk[j] = rk[j * kMergeStep];
        si[j] = ri[j * kMergeStep];
    }
    __syncthreads();
    const int nruns = (m + kRun - 1) / kRun;
    const int lane = threadIdx.x & 31;
    const int wpb = blockDim.x >> 5;
    constexpr int kSpr = kRun / kMergeStep;  // samples per run
    for (int e = blockIdx.x * wpb + (threadIdx.x >> 5); e < m; e += gridDim.x * wpb) {
        const kr_key x = rk[e];
        const int32_t xi = ri[e];
        const int own = e / kRun;
        int c = 0;
        for (int r = lane; r < nruns; r += 32) {
            if (r == own) continue;
            const int r0 = r * kRun, len = min(kRun, m - r0);
            const int nsr = (len + kMergeStep - 1) / kMergeStep;
            // samples of run r smaller than x
            int lo = 0, hi = nsr;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (pair_gt(x, xi, sk[r * kSpr + mid], si[r * kSpr + mid])) lo = mid + 1;
                else hi = mid;
            }
            if (lo == 0) continue;
            const int w0 = r0 + (lo - 1) * kMergeStep;  // the last sample below x
            int cnt = (lo - 1) * kMergeStep + 1;
#pragma unroll
            for (int t = 1; t < kMergeStep; t++) {
                const int q = w0 + t;
                if (q < r0 + len && q < r0 + lo * kMergeStep)
                    cnt += pair_gt(x, xi, rk[q], ri[q]) ? 1 : 0;
            }
            c += cnt;
        }
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

#ifndef KR_ADMIT_VEC
#define KR_ADMIT_VEC 0  // 1: four requests per thread (k_admit_dig)
#endif
#ifndef KR_MERGE_SAMPLED
#define KR_MERGE_SAMPLED 0  // 1: sample-staged rank merge
#endif
#ifndef KR_GROUP_MIN_RUNS
#define KR_GROUP_MIN_RUNS 16  // more runs than this (4k pairs): grouped rank-merge passes
#endif
// KR_MERGE_UNSAMPLED=1: the plain binary-search merge (A/B measurements).
static bool merge_unsampled() {
    static bool v = [] {
        const char* e = getenv("KR_MERGE_UNSAMPLED");
        return e && e[0] == '1';
    }();
    return v;
}

// Sorts (keys, idx) with n elements (keys/idx may alias workspace buffer 0).
static int sort_pairs(const Workspace& w, const kr_key* keys, const int32_t* idx,
                      const unsigned int* count_dev, int64_t n, int32_t* out_idx, kr_key* out_keys,
                      const unsigned long long* stats_dev, cudaStream_t st,
                      const SmallAdmitArgs* ap = nullptr) {
    // ap: the small-fleet admission applied by the final sort stage from the
    // ranks it computes (no separate apply pass); n <= kRunSortMax only
    const SmallAdmitArgs av = ap ? *ap : SmallAdmitArgs{};
    const int apply = ap ? 1 : 0;
    if (n <= kRunSortMax) {
        const int m = static_cast<int>(n);
        const kr_key* sk = keys;
        const int32_t* si = idx;
        // runs are written to the sort ping-pong buffer not holding the input
        kr_key* rk = keys == w.skeys[1] ? w.skeys[0] : w.skeys[1];
        int32_t* ri = keys == w.skeys[1] ? w.sidx[0] : w.sidx[1];
        // more than KR_GROUP_MIN_RUNS runs: grouped merge passes (both outputs
        // given), G = 8 until at most 8 runs remain, the runs ping-ponging
        // between the outputs and the select's candidate buffers (unused by
        // every sort_pairs caller), landing in out.  At 8k pairs (32 runs) two
        // grouped passes (7 + 3 searches per pair) beat one flat pass of 31
        // L2-resident searches: the bench round 483.8 -> 476.3 us, configs[3]
        // 148.7 -> 137.7 us (tools/ab_configs.sh); the flat merge stays for
        // at most 16 runs.
        static const bool grouped_off = std::getenv("KR_MERGE_FLAT") != nullptr;  // A/B knob
        const int runs0 = (m + kRun - 1) / kRun;
        if (apply && runs0 == 1) {  // one run is the whole order
            launch_pdl(k_run_sort, 1, kRunThreads, st, sk, si, count_dev, m, rk, ri, av, 1);
            return check_launch("run sort (apply)");
        }
        if (!grouped_off && out_idx && out_keys && runs0 > KR_GROUP_MIN_RUNS) {
            int lg[8], P = 0;
            for (int r = runs0; r > 1 && P < 8; P++) {
                int g = 0;
                while ((1 << g) < r && g < 3) g++;
                lg[P] = g;
                r = (r + (1 << g) - 1) >> g;
            }
            kr_key* tk = w.cand[0];
            int32_t* ti = reinterpret_cast<int32_t*>(w.cand[1]);
            // the run sort's target: out when an even number of passes follows
            kr_key* ck = P % 2 == 0 ? out_keys : tk;
            int32_t* ci = P % 2 == 0 ? out_idx : ti;
            launch_pdl(k_run_sort, (m + kRun - 1) / kRun, kRunThreads, st, sk, si, count_dev, m, ck,
                       ci, SmallAdmitArgs{}, 0);
            int L = kRun;
            for (int q = 0; q < P; q++) {
                kr_key* dk = (P - 1 - q) % 2 == 0 ? out_keys : tk;
                int32_t* di = (P - 1 - q) % 2 == 0 ? out_idx : ti;
                const int64_t warps = (static_cast<int64_t>(m) + (32 >> lg[q]) - 1) / (32 >> lg[q]);
                int64_t blocks = (warps + 7) / 8;
                if (blocks > 148 * 64) blocks = 148 * 64;
                launch_pdl(k_run_merge_group, static_cast<unsigned>(blocks), 256, st, ck, ci, count_dev,
                           m, L, lg[q], di, dk, av, apply && q == P - 1 ? 1 : 0);
                ck = dk;
                ci = di;
                L <<= lg[q];
            }
            return check_launch("run sort (grouped merge)", 1 + P);
        }
        launch_pdl(k_run_sort, (m + kRun - 1) / kRun, kRunThreads, st, sk, si, count_dev, m, rk, ri,
                   SmallAdmitArgs{}, 0);
        const int64_t warps = m;
        int64_t blocks = (warps + 7) / 8;
        if (blocks > 148 * 64) blocks = 148 * 64;
        if (KR_MERGE_SAMPLED && !apply && m <= kMergeSampled && !merge_unsampled()) {
            // every CTA stages the samples: a few CTAs per SM, several pairs per warp
            const int64_t cap = static_cast<int64_t>(device_info().sm_count) * 2;
            k_run_merge_sampled<<<static_cast<unsigned>(blocks < cap ? blocks : cap), 256, 0, st>>>(
                rk, ri, count_dev, m, out_idx, out_keys);
        }
        else
            launch_pdl(k_run_merge, static_cast<unsigned>(blocks), 256, st, rk, ri, count_dev, m,
                       out_idx, out_keys, av, apply);
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

// scheduler.py:223-234 applied on the owning shard (kr_apply_placements).
__global__ void k_apply_placements(const int32_t* pos, const int32_t* n_placed, int cap,
                                   int64_t run_len, int rank, const int32_t* cand_idx,
                                   const int64_t* obs, int32_t* skipped, uint8_t* refetch,
                                   int64_t now, int64_t stale) {
    const int n = min(*n_placed, cap);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int64_t p = pos[i];
        if (p / run_len != rank) continue;
        const int32_t r = cand_idx[p % run_len];
        if (skipped) skipped[r] = 0;
        if (refetch) refetch[r] = now - obs[r] > stale;
    }
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
// CTAs per SM of the grid passes: fewer CTAs flush fewer partial histograms
// (global atomics on up to 2^11 bins) and fence fewer times.
#ifndef KR_SEL_CPS
#define KR_SEL_CPS 2
#endif
static int sel_ctas_per_sm(int occ) { return KR_SEL_CPS > 0 && KR_SEL_CPS < occ ? KR_SEL_CPS : occ; }

// Launches the select pipeline: state->kth holds the k-th key (and kth_out,
// when given), w.digits the level-0 digits and state->dstar their boundary bin.
static int select_pipeline(const kr_key* keys, int64_t n, int64_t k,
                           const unsigned long long* key_stats, const Workspace& w,
                           kr_key* kth_out, cudaStream_t st, bool prepared = false) {
    SelState* s = w.state;
    int launches = 2;
    if (!prepared) {  // (prepared: the urgency pass's last CTA did this, kr_urgency_prep)
        k_sel_reset<<<1, 1024, 0, st>>>(s, n, k, key_stats, keys);
        launches++;
    }
    if (!key_stats && !prepared) {
        k_sel_stats<<<grid_stream(n), 256, 0, st>>>(keys, n, s);
        k_sel_digit<<<1, 1, 0, st>>>(s, keys);
        launches += 2;
    }
    static int per_sm_h = sel_ctas_per_sm(occupancy(k_sel_hist0, 256));
    static int per_sm_s = sel_ctas_per_sm(occupancy(k_sel_scatter0, 256));
    launch_pdl(k_sel_hist0, grid_cap(n, 256 * kSelU, per_sm_h), 256, st, keys, n, w.digits, s);
    launch_pdl(k_sel_scatter0, grid_cap(n, 256 * kScatW, per_sm_s), 256, st, keys, n, w.digits, w.cand[0],
                                                                   w.cand[1], s, kth_out);
    return check_launch("select", launches);
}

static int admit_with(const kr_key* keys, int64_t n, int64_t k, const kr_key* kth,
                      const kr_fleet* fleet, const kr_sched* cfg, uint8_t* admitted,
                      uint8_t* refetch, int32_t* edge_idx, kr_key* edge_keys, const Workspace& w,
                      cudaStream_t st, const uint16_t* digits = nullptr);

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
    return select_pipeline(keys, n, k, key_stats, w, kth, st);
}

static int select_admit(const kr_key* keys, int64_t n, int64_t k,
                        const unsigned long long* key_stats, const kr_fleet* fleet,
                        const kr_sched* cfg, uint8_t* admitted, uint8_t* refetch,
                        int32_t* edge_idx, kr_key* edge_keys, kr_key* kth_out, void* ws,
                        size_t ws_bytes, void* stream, bool prepared);

extern "C" int kr_select_admit(const kr_key* keys, int64_t n, int64_t k,
                               const unsigned long long* key_stats, const kr_fleet* fleet,
                               const kr_sched* cfg, uint8_t* admitted, uint8_t* refetch,
                               int32_t* edge_idx, kr_key* edge_keys, kr_key* kth_out, void* ws,
                               size_t ws_bytes, void* stream) {
    return select_admit(keys, n, k, key_stats, fleet, cfg, admitted, refetch, edge_idx, edge_keys,
                        kth_out, ws, ws_bytes, stream, false);
}

extern "C" int kr_select_admit_prepared(const kr_key* keys, int64_t n, int64_t k,
                                        const kr_fleet* fleet, const kr_sched* cfg,
                                        uint8_t* admitted, uint8_t* refetch, int32_t* edge_idx,
                                        kr_key* edge_keys, kr_key* kth_out, void* ws,
                                        size_t ws_bytes, void* stream) {
    return select_admit(keys, n, k, nullptr, fleet, cfg, admitted, refetch, edge_idx, edge_keys,
                        kth_out, ws, ws_bytes, stream, true);
}

static int select_admit(const kr_key* keys, int64_t n, int64_t k,
                        const unsigned long long* key_stats, const kr_fleet* fleet,
                        const kr_sched* cfg, uint8_t* admitted, uint8_t* refetch,
                        int32_t* edge_idx, kr_key* edge_keys, kr_key* kth_out, void* ws,
                        size_t ws_bytes, void* stream, bool prepared) {
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
        // the sort's last stage applies the admission (rank < k) itself
        return sort_pairs(w, keys, nullptr, nullptr, n, w.sidx[0], w.skeys[0], nullptr, st, &a);
    }
    Workspace w = carve(ws, n);
    int e = select_pipeline(keys, n, k, key_stats, w, kth_out, st, prepared);
    if (e) return e;
    return admit_with(keys, n, k, &w.state->kth, fleet, cfg, admitted, refetch, edge_idx,
                      edge_keys, w, st, w.digits);
}

// Admission pass + (optional) ordered gather of the admitted set.
static int admit_with(const kr_key* keys, int64_t n, int64_t k, const kr_key* kth,
                      const kr_fleet* fleet, const kr_sched* cfg, uint8_t* admitted,
                      uint8_t* refetch, int32_t* edge_idx, kr_key* edge_keys, const Workspace& w,
                      cudaStream_t st, const uint16_t* digits) {
    const bool gather = edge_idx || edge_keys;
    // after a select the gather state was reset by k_sel_reset
    const bool init = gather && !digits;
    if (init) k_admit_init<<<1, 32, 0, st>>>(w.state);
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
    a.digits = digits;
    if (KR_ADMIT_VEC && digits && kth && k > 0) {
        static int per_sm = occupancy(k_admit_dig, 256);
        k_admit_dig<<<grid_cap(n, 256 * 4, per_sm), 256, 0, st>>>(a);
    } else {
        static int per_sm = occupancy(k_admit, 256);
        launch_pdl(k_admit, grid_cap(n, 256, per_sm), 256, st, a);
    }
    int e = check_launch("k_admit", init ? 2 : 1);
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
    k_sel_reset<<<1, 1024, 0, st>>>(w.state, n, 0, nullptr, keys);
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

extern "C" int kr_apply_placements(const int32_t* pos, const int32_t* n_placed, int64_t cap,
                                   int64_t run_len, int32_t rank, const int32_t* cand_idx,
                                   const kr_fleet* fleet, const kr_sched* cfg, uint8_t* refetch,
                                   void* stream) {
    if (cap < 0 || cap > INT32_MAX || run_len < 1 || rank < 0 || !n_placed) return KR_EINVAL;
    if (cap == 0) return KR_OK;
    if (!pos || !cand_idx || !fleet || (refetch && !cfg)) return KR_EINVAL;
    const int blocks = static_cast<int>((cap + 255) / 256);
    k_apply_placements<<<blocks, 256, 0, as_stream(stream)>>>(
        pos, n_placed, static_cast<int>(cap), run_len, rank, cand_idx, fleet->obs_captured_at,
        fleet->skipped, refetch, cfg ? cfg->now : 0, cfg ? cfg->stale_threshold : 0);
    return check_launch("kr_apply_placements");
}
