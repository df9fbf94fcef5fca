// kr_horizon.cu -- step 1 of the decision core: execution-horizon selection.
//
//   k_horizon_confidence  horizon.py:108-132  confidence-threshold policy over the
//                         [K, N] refinement-update magnitudes of every round
//   k_horizon_divergence  workload.py:461-496 per-timestep cosine divergence
//                         between each new chunk (S samples) and the unexecuted
//                         overlap of the previous chunk, reduced to the longest
//                         prefix that stays at or above the similarity threshold
//
// Both are HBM-bound streaming kernels over fleet-major tensors: each robot's
// rows are one contiguous byte range, tiles of TR robots are moved into shared
// memory by the TMA engine (kr_stream.cuh), and one thread scores one
// (robot, column) or (robot, sample, action) item in fp64 with the reference's
// exact evaluation order.  The per-robot first-trip index is a shared-memory
// atomicMin, which is the parallel form of numpy's argmax / the early-exit loop.
#include <climits>
#include <cmath>
#include <cstring>
#include <type_traits>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <unordered_map>

#include "kr_common.cuh"
#include "kr_host.cuh"
#include "kr_stream.cuh"

namespace kr {

// ---------------------------------------------------------------------------
// Confidence threshold (horizon.py:108-132)
// ---------------------------------------------------------------------------
// Bit-exact fp64 decision of one column: u[:-1].mean(axis=0) is a
// sequential column add for N >= 2 and numpy's pairwise summation when the
// reduction collapses (N == 1); the trip test is a strict '>'.  Out of line:
// it runs only for columns the fp32 filter leaves undecided.
template <typename T>
__device__ __noinline__ bool conf_exact(const T* col, int K, int N, double opt) {
    const int K1 = K - 1;
    double sum;
    if (N >= 2) {
        sum = to_f64(col[0]);
        for (int k = 1; k < K1; k++) sum = dadd(sum, to_f64(col[static_cast<size_t>(k) * N]));
    } else {
        auto a = [col](int64_t k) { return to_f64(col[k]); };
        sum = np_pairwise_sum(a, 0, K1);
    }
    const double m = ddiv(sum, static_cast<double>(K1));
    return to_f64(col[static_cast<size_t>(K1) * N]) > dmul(opt, m);
}

template <typename T, int KC, int VC>
struct ConfWork {
    static constexpr int kVC = VC;
    int K, N, TR, hmin, rounds;
    double opt;   // 1.0 + threshold, rounded on the host as Python does
    float c1;     // (float)(opt / (K - 1)): the fp32 filter's mean-and-scale factor
    float up, dn; // 1 +/- (K + 8) * 2^-24: the fp32 filter's decision margins
    double c1d, upd, dnd;  // fp64 filter: opt / (K - 1), 1 +/- 2^-49
    int32_t* H;
    uint32_t* flags;
    int* first;                  // [kMaxStages][TR] first tripping column per robot
    int rr_q[kMaxRounds];        // this thread's robot slot per round (-1: none)
    int n_q[kMaxRounds];         // ... and first column (VC consecutive columns per item)

    __device__ void setup(int threads) {
        const int items = N / VC;
        for (int q = 0; q < kMaxRounds; q++) {
            const int j = threadIdx.x + q * threads;
            const bool ok = q < rounds && j < TR * items && static_cast<int>(threadIdx.x) < threads;
            rr_q[q] = ok ? j / items : -1;
            n_q[q] = ok ? (j - (j / items) * items) * VC : 0;
        }
    }

    // Exact pre-decision of `f > opt * mean` from the column sum in the storage
    // type, with the mean and the scale folded into one factor (c1 / c1d).
    // fp32: all terms are non-negative, so the fp32 threshold sum * c1 is within
    // (K + 8) * 2^-24 of the exact one relative (up/dn = 1 -/+ that margin).
    // fp64: the sum is the exact path's own sequential sum (N >= 2), so only the
    // folded factor differs: 4 roundings, margin 2^-49.  Branch-free: returns
    // the trip bit and sets `und` for columns it cannot decide (threshold out of
    // range, or within the margin), which take the bit-exact fp64 path.
    // f == 0 never trips (thr >= 0); an exact zero mean trips on any f > 0.
    __device__ __forceinline__ static float add_rn(float a, float b) { return __fadd_rn(a, b); }
    __device__ __forceinline__ static double add_rn(double a, double b) { return __dadd_rn(a, b); }

    __device__ __forceinline__ bool filter(T sf, T fin, bool& und) const {
        bool hi, lo, in_range;
        if constexpr (sizeof(T) == 4) {
            const float thr = __fmul_rn(sf, c1);
            hi = fin > __fmul_rn(thr, up);
            lo = fin < __fmul_rn(thr, dn);
            in_range = thr >= 1e-30f && thr <= 1e30f;
        } else {
            const double thr = __dmul_rn(sf, c1d);
            hi = fin > __dmul_rn(thr, upd);
            lo = fin < __dmul_rn(thr, dnd);
            in_range = thr >= 1e-300 && thr <= 1e300 && N >= 2;  // N == 1: pairwise order
        }
        const bool zero_mean = sf == T(0);
        und = !(fin == T(0) || zero_mean || (in_range && (hi || lo)));
        return hi;
    }

    __device__ __forceinline__ bool exact(const T* col) const { return conf_exact(col, K, N, opt); }

    // Sign/exponent word of a value: a non-negative finite value (+0 included)
    // has it below kBad, so one unsigned max over a column group proves the
    // group valid; otherwise the exact isfinite / '< 0' checks run.
    static constexpr uint32_t kBad = sizeof(T) == 4 ? 0x7f800000u : 0x7ff00000u;
    __device__ __forceinline__ static uint32_t sexp(T x) {
        if constexpr (sizeof(T) == 4) return __float_as_uint(x);
        else return static_cast<uint32_t>(__double_as_longlong(x) >> 32);
    }
    __device__ __forceinline__ static uint32_t check(T x) {
        uint32_t fl = 0;
        if (!isfinite(x)) fl |= KR_FLAG_NONFINITE;
        if (x < T(0)) fl |= KR_FLAG_NEGATIVE;
        return fl;
    }

    // VC consecutive columns of row k (vector load when VC > 1: N % VC == 0
    // and the tile base is aligned, checked on the host)
    __device__ __forceinline__ static void load_row(const T* row, T (&x)[VC]) {
        if constexpr (VC == 1) {
            x[0] = row[0];
        } else if constexpr (sizeof(T) == 4 && VC == 2) {
            const float2 v = *reinterpret_cast<const float2*>(row);
            x[0] = v.x; x[1] = v.y;
        } else if constexpr (sizeof(T) == 4 && VC == 4) {
            const float4 v = *reinterpret_cast<const float4*>(row);
            x[0] = v.x; x[1] = v.y; x[2] = v.z; x[3] = v.w;
        } else {
#pragma unroll
            for (int v = 0; v < VC; v += 2) {
                const double2 d = *reinterpret_cast<const double2*>(row + v);
                x[v] = d.x; x[v + 1] = d.y;
            }
        }
    }

    __device__ __forceinline__ void tile(const TileView& v, int64_t, int nr, int slot) {
        const T* u = reinterpret_cast<const T*>(v.seg[0]);
        int* f = first + slot * TR;
        uint32_t fl = 0;
        const int Kr = KC > 0 ? KC : K;
#pragma unroll
        for (int q = 0; q < kMaxRounds; q++) {
            if (q >= rounds) break;
            const int rr = rr_q[q];
            const bool valid = rr >= 0 && rr < nr;
            int idx = INT_MAX;
            if (valid) {
                const int n0 = n_q[q];
                const T* col = u + static_cast<size_t>(rr) * Kr * N + n0;
                // one pass over the columns: validation (horizon.py:47-50) + filter sums
                T sf[VC], fin[VC];
                uint32_t mx = 0;
                bool bad = false;
                if constexpr (KC > 0) {
                    T x[KC][VC];
#pragma unroll
                    for (int k = 0; k < KC; k++) load_row(col + static_cast<size_t>(k) * N, x[k]);
#pragma unroll
                    for (int k = 0; k < KC; k++)
#pragma unroll
                        for (int c = 0; c < VC; c++) mx = max(mx, sexp(x[k][c]));
                    if (mx >= kBad) {
#pragma unroll
                        for (int k = 0; k < KC; k++)
#pragma unroll
                            for (int c = 0; c < VC; c++) fl |= check(x[k][c]);
                        bad = true;
                    }
#pragma unroll
                    for (int c = 0; c < VC; c++) {
                        sf[c] = x[0][c];
#pragma unroll
                        for (int k = 1; k < KC - 1; k++) sf[c] = add_rn(sf[c], x[k][c]);
                        fin[c] = x[KC - 1][c];
                    }
                } else {
                    for (int k = 0; k < Kr; k++) {
                        T x[VC];
                        load_row(col + static_cast<size_t>(k) * N, x);
#pragma unroll
                        for (int c = 0; c < VC; c++) {
                            mx = max(mx, sexp(x[c]));
                            if (k == 0) sf[c] = x[c];
                            else if (k < Kr - 1) sf[c] = add_rn(sf[c], x[c]);
                            else fin[c] = x[c];
                        }
                    }
                    if (mx >= kBad) {
                        for (int k = 0; k < Kr; k++)
                            for (int c = 0; c < VC; c++) fl |= check(col[static_cast<size_t>(k) * N + c]);
                        bad = true;
                    }
                }
#pragma unroll
                for (int c = VC - 1; c >= 0; c--) {
                    bool und;
                    bool t = filter(sf[c], fin[c], und);
                    if (und || bad) t = exact(col + c);
                    if (t) idx = n0 + c;
                }
            }
            first_flag(f, valid ? rr : -1, valid ? rr : -1, idx != INT_MAX, idx);
        }
        if (fl && flags) atomicOr(flags, fl);
    }

    __device__ __forceinline__ void finish(int64_t r0, int nr, int slot, int t, int nt) {
        int* f = first + slot * TR;
        for (int rr = t; rr < nr; rr += nt) {
            int h = f[rr] < N ? f[rr] : N;  // argmax of trips, or N
            h = h > hmin ? h : hmin;
            H[r0 + rr] = h < N ? h : N;
            f[rr] = INT_MAX;
        }
    }
};

// several columns per thread need more than 64 registers: cap the block at 512
template <int VC>
constexpr int conf_max_threads() { return VC == 1 ? kStreamThreads : 512; }

template <typename T, int KC, int VC, bool kStaged>
__global__ void __launch_bounds__(conf_max_threads<VC>()) k_horizon_confidence(StreamPlan p, ConfWork<T, KC, VC> w) {
    extern __shared__ __align__(128) unsigned char smem[];
    w.first = reinterpret_cast<int*>(smem + stream_aux_offset());
    for (int i = threadIdx.x; i < kMaxStages * w.TR; i += blockDim.x) w.first[i] = INT_MAX;
    w.setup(p.threads);
    __syncthreads();
    stream_run<kStaged>(p, smem, w);
}

// ---------------------------------------------------------------------------
// Divergence horizon (workload.py:461-496), S-sample ensembles, ragged rows
// ---------------------------------------------------------------------------
// SL ("samples looped", S > 1): one thread per (robot, action) scores all S
// samples against the reference row it loads once (kept in registers for
// small D); the robot's horizon is the first action where ANY sample falls
// below the threshold, so one first-trip reduction per action suffices.
template <typename T, int DC, bool SL = false>
struct DivWork {
    int S, Lp, Lc, D, TR, rounds;
    bool has_off, has_lp, has_lc;  // per-robot arrays present (segment slots 2, 3, 4)
    double thr;
    int32_t* H;
    double* cos;
    float thr_f, margin;
    int* first;                   // [kMaxStages][TR] first failing action per robot
    int* lim;                     // [kMaxStages][TR] prefix limit per robot
    int rr_q[kMaxRounds], s_q[kMaxRounds], i_q[kMaxRounds];

    __device__ void setup(int threads) {
        const int per = SL ? Lc : S * Lc;
        for (int q = 0; q < kMaxRounds; q++) {
            const int j = threadIdx.x + q * threads;
            const bool ok = q < rounds && j < TR * per && static_cast<int>(threadIdx.x) < threads;
            const int rr = ok ? j / per : -1;
            const int rem = ok ? j - rr * per : 0;
            rr_q[q] = rr;
            s_q[q] = rem / Lc;
            i_q[q] = rem - (rem / Lc) * Lc;
        }
    }

    __device__ __forceinline__ int2 meta(const TileView& v, int rr) const {
        int o = has_off ? reinterpret_cast<const int32_t*>(v.seg[2])[rr] : 0;
        o = o < 0 ? 0 : o;
        if (!has_lp && !has_lc) {  // common case: only the overlap offset varies
            const int lr = Lp - o;
            return make_int2(o, lr < Lc ? (lr < 0 ? 0 : lr) : Lc);
        }
        int lp = has_lp ? reinterpret_cast<const int32_t*>(v.seg[3])[rr] : Lp;
        int lc = has_lc ? reinterpret_cast<const int32_t*>(v.seg[4])[rr] : Lc;
        lp = lp > Lp ? Lp : lp;
        lc = lc > Lc ? Lc : (lc < 0 ? 0 : lc);
        int lr = lp - o;
        lr = lr < 0 ? 0 : lr;
        return make_int2(o, lr < lc ? lr : lc);
    }

    // one (robot, action): every sample against the reference row
    __device__ __forceinline__ bool fail_any(const T* a0, const T* b, double* cp) const {
        const int D_ = DC > 0 ? DC : D;
        const size_t sstride = static_cast<size_t>(Lc) * D_;
        bool fail = false;
        if constexpr (DC > 0 && DC < 16) {
            float y[DC], yy = 0.f;
#pragma unroll
            for (int e = 0; e < DC; e++) {
                y[e] = static_cast<float>(b[e]);
                yy = __fmaf_rn(y[e], y[e], yy);
            }
            for (int s = 0; s < S; s++) {
                const T* a = a0 + s * sstride;
                double* c_out = cp ? cp + static_cast<size_t>(s) * Lc : nullptr;
                int pass = -1;
                if (!c_out) {
                    float xx = 0.f, xy = 0.f;
#pragma unroll
                    for (int e = 0; e < DC; e++) {
                        const float x = static_cast<float>(a[e]);
                        xx = __fmaf_rn(x, x, xx);
                        xy = __fmaf_rn(x, y[e], xy);
                    }
                    pass = cos_filter_decide(xx, yy, xy, thr_f, margin);
                }
                if (pass < 0) {
                    const double c = cosine_skx_fixed<DC>(a, b);
                    pass = !(c < thr);
                    if (c_out) *c_out = c;
                }
                if (!pass) {
                    fail = true;
                    if (!cp) break;
                }
            }
        } else {
            for (int s = 0; s < S; s++) {
                const T* a = a0 + s * sstride;
                double* c_out = cp ? cp + static_cast<size_t>(s) * Lc : nullptr;
                int pass = -1;
                if (!c_out) {
                    if constexpr (DC > 0)
                        pass = cos_filter_fixed<DC>(a, b, thr_f, margin);
                    else
                        pass = cos_filter(a, b, D_, thr_f, margin);
                }
                if (pass < 0) {
                    double c;
                    if constexpr (DC > 0)
                        c = cosine_skx_fixed<DC>(a, b);
                    else
                        c = cosine_skx(a, b, D_);
                    pass = !(c < thr);
                    if (c_out) *c_out = c;
                }
                if (!pass) {
                    fail = true;
                    if (!cp) break;
                }
            }
        }
        return fail;
    }

    __device__ __forceinline__ void tile(const TileView& v, int64_t r0, int nr, int slot) {
        const T* prev = reinterpret_cast<const T*>(v.seg[0]);
        const T* cand = reinterpret_cast<const T*>(v.seg[1]);
        int* f = first + slot * TR;
        int* lm = lim + slot * TR;
        const int D_ = DC > 0 ? DC : D;
        if constexpr (SL) {
#pragma unroll
            for (int q = 0; q < kMaxRounds; q++) {
                if (q >= rounds) break;
                const int rr = rr_q[q], i = i_q[q];
                const bool valid = rr >= 0 && rr < nr;
                bool fail = false;
                if (valid) {
                    const int2 m = meta(v, rr);
                    if (i == 0) lm[rr] = m.y;
                    double* cp = cos ? cos + static_cast<size_t>(r0 + rr) * S * Lc + i : nullptr;
                    if (i < m.y) {
                        const T* a0 = cand + (static_cast<size_t>(rr) * S * Lc + i) * D_;
                        const T* b = prev + (static_cast<size_t>(rr) * Lp + m.x + i) * D_;
                        fail = fail_any(a0, b, cp);
                    } else if (cp) {
                        for (int s = 0; s < S; s++)
                            cp[static_cast<size_t>(s) * Lc] = __longlong_as_double(0x7ff8000000000000LL);
                    }
                }
                first_flag(f, valid ? rr : -1, valid ? rr : -1, fail, i);
            }
            return;
        }
#pragma unroll
        for (int q = 0; q < kMaxRounds; q++) {
            if (q >= rounds) break;
            const int rr = rr_q[q], s = s_q[q], i = i_q[q];
            const bool valid = rr >= 0 && rr < nr;
            bool fail = false;
            if (valid) {
                const int2 m = meta(v, rr);
                if (i == 0 && s == 0) lm[rr] = m.y;
                double* cp = cos ? cos + (static_cast<size_t>(r0 + rr) * S + s) * Lc + i : nullptr;
                if (i < m.y) {
                    const T* a = cand + (static_cast<size_t>(rr * S + s) * Lc + i) * D_;
                    const T* b = prev + (static_cast<size_t>(rr) * Lp + m.x + i) * D_;
                    int pass = -1;
                    if (!cp) {
                        if constexpr (DC > 0)
                            pass = cos_filter_fixed<DC>(a, b, thr_f, margin);
                        else
                            pass = cos_filter(a, b, D_, thr_f, margin);
                    }
                    if (pass < 0) {
                        double c;
                        if constexpr (DC > 0)
                            c = cosine_skx_fixed<DC>(a, b);
                        else
                            c = cosine_skx(a, b, D_);
                        pass = !(c < thr);
                        if (cp) *cp = c;
                    }
                    fail = !pass;  // the first action below threshold ends the prefix
                } else if (cp) {
                    *cp = __longlong_as_double(0x7ff8000000000000LL);  // NaN past the limit
                }
            }
            first_flag(f, valid ? rr : -1, valid ? rr * S + s : -1, fail, i);
        }
    }

    __device__ __forceinline__ void finish(int64_t r0, int nr, int slot, int t, int nt) {
        int* f = first + slot * TR;
        const int* lm = lim + slot * TR;
        for (int rr = t; rr < nr; rr += nt) {
            H[r0 + rr] = f[rr] < lm[rr] ? f[rr] : lm[rr];
            f[rr] = INT_MAX;
        }
    }
};

// Small-D variants keep every operand in < 64 registers and may use 1024-thread
// CTAs; D >= 16 (and runtime D) need the 32 fp64 OpenBLAS accumulators, so
// their CTAs are capped at 256 threads (255 registers available).
template <int DC>
constexpr int div_max_threads() { return (DC > 0 && DC < 16) ? kStreamThreads : 256; }

template <typename T, int DC, bool kStaged, bool SL = false>
__global__ void __launch_bounds__(div_max_threads<DC>()) k_horizon_divergence(StreamPlan p,
                                                                             DivWork<T, DC, SL> w) {
    extern __shared__ __align__(128) unsigned char smem[];
    w.first = reinterpret_cast<int*>(smem + stream_aux_offset());
    w.lim = w.first + kMaxStages * w.TR;
    for (int i = threadIdx.x; i < kMaxStages * w.TR; i += blockDim.x) w.first[i] = INT_MAX;
    w.setup(p.threads);
    __syncthreads();
    stream_run<kStaged>(p, smem, w);
}

// ---------------------------------------------------------------------------
// Threshold sweep (horizon.py:135-151 sweep_thresholds, cli.py:109-140
// cmd_pareto): C policy configurations decided over the same rounds in ONE
// pass over U.
//
// The column statistics (sum, final) do not depend on the configuration, and
// the trip test f > fl(p * m) is monotone in p = 1 + t: with the confidence
// configurations sorted by p, the ones a column trips form a prefix [0, j_n).
// One filter per column gives j_n (fast exits for "none" / "all", otherwise a
// binary search over the sorted factors with the K1 margins, and the
// bit-exact fp64 mean when the margins cannot decide).
//
// A warp owns one robot at a time (lane = VC adjacent columns, chunks of
// 32 * VC columns).  With M_n = max_{n' <= n} j_n' (a warp max-scan carried
// across chunks), configuration c's horizon is the first n with M_n > c, so
// the column where M steps from a to b is the horizon of exactly the
// configurations [a, b) -- one lane per step, no per-configuration loop.  The
// per-configuration sums are accumulated as a difference array over the
// sorted slots (D[a] += n, D[b] -= n; never-tripped slots [M_last, Cc) get
// N), plus a correction F[c] += hmin_c - n for the rare steps below a
// configuration's min_horizon floor.  S_c = prefix_sum(D)[c] + F[c] at the end
// of the CTA; the optional H[c][r] output writes every decision.
// ---------------------------------------------------------------------------
constexpr int kSweepMaxCfg = 64;
constexpr int kSweepPad = 128;  // search tables: a power of two > Cc, padded with +inf
constexpr int kSweepLut = 2048; // ratio buckets

struct SweepCfg {
    int32_t C, Cc;                       // configurations, confidence ones (sorted first)
    int32_t maxcap;                      // max over confidence slots of min(min_horizon, N)
    int32_t half;                        // P / 2: first step of the branch-free search
    int32_t lut_n, lut_shift;            // ratio buckets (0: none), bits dropped per bucket
    uint64_t lut_lo, lut_hi;             // storage-type bit patterns of the bucketed ratio range
    double sfmin, sfmax;                 // column sums whose ratio stays a normal number
    int32_t orig[kSweepMaxCfg];          // sorted slot -> caller's configuration index
    int32_t hcap[kSweepMaxCfg];          // confidence: min(min_horizon, N); static: min(static_h, N)
    double p[kSweepMaxCfg];              // 1 + t, ascending (confidence slots)
    double rh[kSweepPad], rl[kSweepPad]; // ratio bounds (1 + t) / (K - 1) * (1 +/- margin), outward
    uint16_t lut[kSweepLut];             // bucket -> tripping slots, 0xFFFF: undecided
};

// shared copies of the per-configuration tables (indexed per lane)
struct SweepTables {
    double rhd[kSweepPad], rld[kSweepPad];
    float rh[kSweepPad], rl[kSweepPad];
    double p[kSweepMaxCfg];
    int32_t orig[kSweepMaxCfg];
    int32_t hcap[kSweepMaxCfg];
    // per-CTA sums stay below 2^32: R * N elements fit in HBM, so a CTA's share
    // (R / grid robots, N columns, horizons <= N) is < 2^32; checked on the host
    uint32_t D[kSweepMaxCfg + 1];  // difference array of the per-slot sums (mod 2^32)
    uint32_t F[kSweepMaxCfg];      // min_horizon floor corrections
    uint16_t lut[kSweepLut];
};

// Bit-exact count of tripping confidence configurations for one column.
template <typename T>
__device__ __noinline__ int sweep_exact(const T* col, int K, int N, const double* p, int Cc) {
    const int K1 = K - 1;
    double sum;
    if (N >= 2) {
        sum = to_f64(col[0]);
        for (int k = 1; k < K1; k++) sum = dadd(sum, to_f64(col[static_cast<size_t>(k) * N]));
    } else {
        auto a = [col](int64_t k) { return to_f64(col[k]); };
        sum = np_pairwise_sum(a, 0, K1);
    }
    const double m = ddiv(sum, static_cast<double>(K1));
    const double f = to_f64(col[static_cast<size_t>(K1) * N]);
    int lo = 0, hi = Cc;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (f > dmul(p[mid], m)) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

template <typename T, int KC, int VC>
struct SweepWork {
    using CW = ConfWork<T, KC, VC>;
    using Elem = T;
    static constexpr int kVC = VC;
    int K, N, TR, C, Cc, maxcap, half;
    int cw;                      // consumer warps (robots are dealt round-robin to them)
    int lut_n, lut_shift;
    uint64_t lut_lo, lut_hi;
    T sfmin, sfmax;
    int32_t* H;                  // [C][R] (nullable)
    unsigned long long* sums;    // [C]
    uint32_t* flags;
    int64_t R;
    SweepTables* tab;            // shared

    __device__ void setup(int) {}

    // Number of confidence configurations the column trips, or -1 when the
    // margins cannot decide it.  The column's ratio f / sum (one approximate
    // reciprocal) against the slot factors c = (1 + t) / (K - 1): rh[c] / rl[c]
    // widen c by the filter margin (fp32 sum, reciprocal and products:
    // (K + 8) 2^-24; fp64: 2^-49), so ratio > rh[c] is a definite trip and
    // ratio < rl[c] a definite non-trip; both hold for prefixes of the sorted
    // slots.  A bucket table over the ratio's bit pattern answers most columns
    // with one lookup; buckets that straddle a slot bound fall back to a
    // branch-free binary search.  f == 0 never trips; an exact zero mean trips
    // on any f > 0.
    // Branch-free common path: the bucket lookup and the zero rules; `und`
    // marks columns that need search() (ambiguous bucket, sum out of range).
    __device__ __forceinline__ int filter(T sf, T fin, T& rho, bool& und) const {
        using B = typename std::conditional<sizeof(T) == 4, uint32_t, uint64_t>::type;
        B bits;
        if constexpr (sizeof(T) == 4) {
            float r;
            asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(sf));  // <= 1 ulp, sf normal
            rho = __fmul_rn(fin, r);
            bits = __float_as_uint(rho);
        } else {
            rho = __dmul_rn(fin, __drcp_rn(sf));
            bits = static_cast<uint64_t>(__double_as_longlong(rho));
        }
        const B lo = static_cast<B>(lut_lo), hi = static_cast<B>(lut_hi);
        const bool below = bits < lo, above = bits >= hi;
        const uint32_t off = below || above ? 0u : static_cast<uint32_t>((bits - lo) >> lut_shift);
        const unsigned e = tab->lut[off];
        int j = below ? 0 : (above ? Cc : static_cast<int>(e));
        und = !below && !above && e == 0xFFFFu;
        und = und || !(sf >= sfmin && sf <= sfmax);
        if (sf == T(0)) { j = Cc; und = false; }
        if (fin == T(0)) { j = 0; und = false; }
        return j;
    }

    // ambiguous bucket: branch-free binary search over the slot bounds
    __device__ __forceinline__ int search(T sf, T rho) const {
        if (!(sf >= sfmin && sf <= sfmax)) return -1;
        const T* rh;
        const T* rl;
        if constexpr (sizeof(T) == 4) { rh = tab->rh; rl = tab->rl; }
        else { rh = tab->rhd; rl = tab->rld; }
        int pos = 0;
        for (int st = half; st > 0; st >>= 1)
            if (rho > rh[pos + st - 1]) pos += st;
        if (pos == Cc || rho < rl[pos]) return pos;
        return -1;
    }

    // configurations [a, b) take horizon n at this robot (a < b)
    __device__ __forceinline__ void step(int a, int b, int n, int64_t r) const {
        atomicAdd(&tab->D[a], static_cast<uint32_t>(n));
        atomicSub(&tab->D[b], static_cast<uint32_t>(n));
        if (n < maxcap)  // below some min_horizon floor (horizon.py:130)
            for (int c = a; c < b; c++) {
                const int cap = tab->hcap[c];
                if (cap > n) atomicAdd(&tab->F[c], static_cast<uint32_t>(cap - n));
            }
        if (H)
            for (int c = a; c < b; c++) {
                const int cap = tab->hcap[c];
                H[static_cast<int64_t>(tab->orig[c]) * R + r] = n > cap ? n : cap;
            }
    }

    __device__ __noinline__ uint32_t check_all(const T* col) const {
        uint32_t fl = 0;
        const int Kr = KC > 0 ? KC : K;
        for (int k = 0; k < Kr; k++)
            for (int c = 0; c < VC; c++) fl |= CW::check(col[k * N + c]);
        return fl;
    }

    __device__ __forceinline__ void tile(const TileView& v, int64_t r0, int nr, int) {
        const T* u = reinterpret_cast<const T*>(v.seg[0]);
        uint32_t fl = 0;
        const int Kr = KC > 0 ? KC : K;
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        if (warp >= cw) return;  // the producer warp's slot in the non-TMA modes
        const int KN = Kr * N;
        for (int rr = warp; rr < nr; rr += cw) {
            const T* rob = u + rr * KN;
            int carry = 0;  // M of the previous chunk's last column
            for (int n0c = 0; n0c < N; n0c += 32 * VC) {
                const int n0 = n0c + lane * VC;
                const bool valid = n0 < N;
                int j[VC];
#pragma unroll
                for (int c = 0; c < VC; c++) j[c] = 0;
                if (valid) {
                    const T* col = rob + n0;
                    T sf[VC], fin[VC];
                    uint32_t mx = 0;
                    if constexpr (KC > 0) {
                        T x[KC][VC];
#pragma unroll
                        for (int k = 0; k < KC; k++) CW::load_row(col + k * N, x[k]);
#pragma unroll
                        for (int k = 0; k < KC; k++)
#pragma unroll
                            for (int c = 0; c < VC; c++) mx = max(mx, CW::sexp(x[k][c]));
#pragma unroll
                        for (int c = 0; c < VC; c++) {
                            sf[c] = x[0][c];
#pragma unroll
                            for (int k = 1; k < KC - 1; k++) sf[c] = CW::add_rn(sf[c], x[k][c]);
                            fin[c] = x[KC - 1][c];
                        }
                    } else {
                        for (int k = 0; k < Kr; k++) {
                            T x[VC];
                            CW::load_row(col + k * N, x);
#pragma unroll
                            for (int c = 0; c < VC; c++) {
                                mx = max(mx, CW::sexp(x[c]));
                                if (k == 0) sf[c] = x[c];
                                else if (k < Kr - 1) sf[c] = CW::add_rn(sf[c], x[c]);
                                else fin[c] = x[c];
                            }
                        }
                    }
                    const bool bad = mx >= CW::kBad;
                    bool und[VC];
                    T rho[VC];
#pragma unroll
                    for (int c = 0; c < VC; c++) {
                        j[c] = filter(sf[c], fin[c], rho[c], und[c]);
                        und[c] = und[c] || bad;
                    }
                    if (bad) fl |= check_all(col);
#pragma unroll
                    for (int c = 0; c < VC; c++)
                        if (und[c]) {
                            int jj = bad ? -1 : search(sf[c], rho[c]);
                            if (jj < 0) jj = sweep_exact(col + c, K, N, tab->p, Cc);
                            j[c] = jj;
                        }
                }
                __syncwarp();
                int jt = carry;
#pragma unroll
                for (int c = 0; c < VC; c++) jt = max(jt, j[c]);
                // inclusive max-scan over the lanes (columns ascend with the lane)
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const int o = __shfl_up_sync(0xffffffffu, jt, d);
                    if (lane >= d) jt = max(jt, o);
                }
                int cur = __shfl_up_sync(0xffffffffu, jt, 1);
                if (lane == 0) cur = carry;
                if (valid && jt > cur) {
#pragma unroll
                    for (int c = 0; c < VC; c++)
                        if (j[c] > cur) {
                            step(cur, j[c], n0 + c, r0 + rr);
                            cur = j[c];
                        }
                }
                carry = __shfl_sync(0xffffffffu, jt, 31);
            }
            // slots never tripped take the whole chunk (>= every floor)
            if (lane == 0 && carry < Cc) {
                atomicAdd(&tab->D[carry], static_cast<uint32_t>(N));
                if (H)
                    for (int c = carry; c < Cc; c++)
                        H[static_cast<int64_t>(tab->orig[c]) * R + r0 + rr] = N;
            }
            if (H)
                for (int c = Cc + lane; c < C; c += 32)
                    H[static_cast<int64_t>(tab->orig[c]) * R + r0 + rr] = tab->hcap[c];
        }
        if (fl && flags) atomicOr(flags, fl);
    }

    __device__ __forceinline__ void finish(int64_t, int, int, int, int) {}
};

constexpr int kSweepThreads = 384;

template <typename T, int KC, int VC, bool kStaged>
__global__ void __launch_bounds__(kSweepThreads, 2) k_horizon_sweep(StreamPlan p,
                                                                         SweepWork<T, KC, VC> w,
                                                                         const __grid_constant__ SweepCfg cfg) {
    extern __shared__ __align__(128) unsigned char smem[];
    w.tab = reinterpret_cast<SweepTables*>(smem + stream_aux_offset());
    for (int i = threadIdx.x; i < w.lut_n; i += blockDim.x) w.tab->lut[i] = cfg.lut[i];
    for (int i = threadIdx.x; i < kSweepPad; i += blockDim.x) {
        w.tab->rhd[i] = cfg.rh[i];
        w.tab->rld[i] = cfg.rl[i];
        w.tab->rh[i] = static_cast<float>(cfg.rh[i]);  // exactly representable (host-rounded)
        w.tab->rl[i] = static_cast<float>(cfg.rl[i]);
        if (i < kSweepMaxCfg) {
            w.tab->p[i] = cfg.p[i];
            w.tab->orig[i] = cfg.orig[i];
            w.tab->hcap[i] = cfg.hcap[i];
            w.tab->F[i] = 0;
        }
        if (i <= kSweepMaxCfg) w.tab->D[i] = 0;
    }
    __syncthreads();
    stream_run<kStaged>(p, smem, w);
    __syncthreads();
    if (threadIdx.x == 0) {  // S_c = prefix_sum(D)[c] + F[c]; static slots once per grid
        uint32_t run = 0;
        for (int c = 0; c < w.Cc; c++) {
            run += w.tab->D[c];
            const uint32_t s = run + w.tab->F[c];
            if (s) atomicAdd(&w.sums[w.tab->orig[c]], static_cast<unsigned long long>(s));
        }
        if (blockIdx.x == 0)
            for (int c = w.Cc; c < w.C; c++)
                atomicAdd(&w.sums[w.tab->orig[c]],
                          static_cast<unsigned long long>(w.R) * static_cast<unsigned long long>(w.tab->hcap[c]));
    }
}

__global__ void k_horizon_static(int64_t R, int32_t h, int32_t* H) {
    for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < R;
         r += int64_t(gridDim.x) * blockDim.x)
        H[r] = h;
}

// ---------------------------------------------------------------------------
// Launch planning
// ---------------------------------------------------------------------------
// Tile shape search.  For each candidate TR (robots per tile) the CTA gets
// ceil(TR * items / rounds) threads (rounds <= 4, a multiple of 32) so every
// thread owns fixed positions.  Residency (CTAs per SM) is bounded by the
// kernel's register count, the 2048-thread limit and shared memory; the TMA
// ring then takes as many stages as fit (up to 8).  Score: idle-lane fraction,
// plus penalties for < 160 KB of TMA bytes in flight per SM (the loaded HBM
// latency times the per-SM share of bandwidth), < 24 resident warps per SM,
// and tiles that cannot be moved by TMA.
static StreamPlan make_plan(int nseg, const void* const* base, const uint64_t* rbytes, int64_t R,
                            int items_per_robot, uint32_t aux_per_robot, int max_threads,
                            int regs_per_thread, int min_rounds = 1, uint32_t aux_fixed = 256,
                            int force_tr = 0) {
    const DeviceInfo& di = device_info();
    StreamPlan p{};
    p.nseg = nseg;
    p.R = R;
    bool base_ok = true;
    for (int g = 0; g < nseg; g++) {
        p.base[g] = static_cast<const unsigned char*>(base[g]);
        p.rbytes[g] = static_cast<uint32_t>(rbytes[g]);
        if (rbytes[g]) base_ok = base_ok && aligned16(base[g]);
    }
    auto stage_bytes = [&](int64_t t) {
        uint64_t b = 0;
        for (int g = 0; g < nseg; g++) b += ((uint64_t)t * rbytes[g] + 127) & ~uint64_t(127);
        return b;
    };
    auto tma_ok = [&](int64_t t) {
        for (int g = 0; g < nseg; g++)
            if ((t * rbytes[g]) % 16) return false;
        return base_ok;
    };
    static const int max_override = std::getenv("KR_PLAN_MAX_THREADS")
                                        ? std::atoi(std::getenv("KR_PLAN_MAX_THREADS")) : 0;
    if (max_override >= 32 && max_override < max_threads) max_threads = max_override;
    static const int rounds_override = std::getenv("KR_PLAN_MIN_ROUNDS")
                                           ? std::atoi(std::getenv("KR_PLAN_MIN_ROUNDS")) : 0;
    if (rounds_override >= 1 && rounds_override <= kMaxRounds) min_rounds = rounds_override;
    const int regs = ((regs_per_thread > 0 ? regs_per_thread : 64) + 7) / 8 * 8;
    const uint64_t smem_sm = static_cast<uint64_t>(di.max_smem_optin) + 1024;  // per-SM pool
    const double kInflightTarget = 160.0 * 1024;
    double best = 1e30;
    for (int64_t t = force_tr > 0 ? force_tr : 1; t <= (force_tr > 0 ? force_tr : 1024); t++) {
        const int64_t items = t * items_per_robot;
        if (items > static_cast<int64_t>(max_threads) * kMaxRounds) break;
        int rounds = static_cast<int>((items + max_threads - 1) / max_threads);
        if (rounds < min_rounds) {
            if (items < static_cast<int64_t>(min_rounds) * 32) continue;
            rounds = min_rounds;
        }
        const int threads = static_cast<int>(((items + rounds - 1) / rounds + 31) / 32 * 32);
        const uint64_t sb = stage_bytes(t);
        const uint64_t aux = (aux_fixed + t * aux_per_robot + 127) & ~uint64_t(127);
        const bool tma = tma_ok(t);
        const int cta = threads + 32;  // + the producer warp
        int per_sm = 65536 / (regs * cta);
        per_sm = per_sm < 2048 / cta ? per_sm : 2048 / cta;
        per_sm = per_sm > 4 ? 4 : per_sm;
        for (; per_sm >= 1; per_sm--) {
            const uint64_t budget = smem_sm / per_sm - 1024 - 128;  // 1 KB reserved per CTA
            if (aux + 2 * sb <= budget) break;
        }
        if (per_sm < 1) continue;
        const uint64_t budget = smem_sm / per_sm - 1024 - 128;
        int stages = static_cast<int>((budget - aux) / sb);
        stages = stages > kMaxStages ? kMaxStages : stages;
        const double inflight = static_cast<double>(per_sm) * (stages - 1) * sb;
        const double warps = per_sm * cta / 32.0;
        double score = 1.0 - static_cast<double>(items) / (static_cast<double>(rounds) * threads);
        if (inflight < kInflightTarget) score += 0.5 * (1.0 - inflight / kInflightTarget);
        if (warps < 24.0) score += 0.2 * (1.0 - warps / 24.0);
        if (!tma) score += 1.0;
        if (score < best - 1e-9) {
            best = score;
            p.TR = static_cast<int>(t);
            p.threads = threads;
            p.rounds = rounds;
            p.stages = stages;
            p.mode = tma ? kModeBulk : kModePlain;
        }
    }
    if (best > 1e29) {  // robot larger than two stages of shared memory: score from global
        p.TR = 1;
        p.rounds = static_cast<int>((items_per_robot + max_threads - 1) / max_threads);
        if (p.rounds > kMaxRounds) p.rounds = kMaxRounds;  // caller guarantees it fits
        p.threads = static_cast<int>(((items_per_robot + p.rounds - 1) / p.rounds + 31) / 32 * 32);
        p.stages = 1;
        p.mode = kModeDirect;
        p.aux_bytes = aux_fixed + aux_per_robot;
        p.stage_bytes = 0;
        return p;
    }
    p.aux_bytes = static_cast<uint32_t>(aux_fixed + p.TR * aux_per_robot);
    uint32_t off = 0;
    for (int g = 0; g < nseg; g++) {
        p.soff[g] = off;
        off += static_cast<uint32_t>(((uint64_t)p.TR * rbytes[g] + 127) & ~uint64_t(127));
    }
    p.stage_bytes = off;
    if (p.mode == kModePlain) p.stages = 1;
    return p;
}

// Per-kernel launch facts, cached so that repeated (and CUDA-graph-captured)
// launches make no attribute / occupancy queries.
struct KernelFacts {
    int regs = -1;
    int smem_set = 0;
    int occ_threads = 0, occ_smem = -1, occ_blocks = 0;
};
static std::mutex g_facts_mu;
static std::unordered_map<const void*, KernelFacts> g_facts;

template <class K>
static int kernel_regs(K kern) {
    std::lock_guard<std::mutex> lock(g_facts_mu);
    KernelFacts& f = g_facts[reinterpret_cast<const void*>(kern)];
    if (f.regs < 0) {
        cudaFuncAttributes a{};
        f.regs = cudaFuncGetAttributes(&a, kern) == cudaSuccess ? a.numRegs : 64;
    }
    return f.regs;
}

template <class Work, class KStaged, class KDirect, class... Extra>
static int launch_stream(KStaged kstaged, KDirect kdirect, const StreamPlan& p, const Work& w,
                         cudaStream_t st, const char* name, int max_sms = 0,
                         const Extra&... extra) {
    size_t smem = stream_smem_bytes(p);
    auto go = [&](auto kern) -> int {
        int per_sm = 0;
        {
            std::lock_guard<std::mutex> lock(g_facts_mu);
            KernelFacts& f = g_facts[reinterpret_cast<const void*>(kern)];
            if (f.smem_set < static_cast<int>(smem)) {
                KR_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 static_cast<int>(smem)));
                f.smem_set = static_cast<int>(smem);
            }
            if (f.occ_threads != p.threads || f.occ_smem != static_cast<int>(smem)) {
                KR_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&f.occ_blocks, kern,
                                                                          p.threads + 32, smem));
                f.occ_threads = p.threads;
                f.occ_smem = static_cast<int>(smem);
            }
            per_sm = f.occ_blocks;
        }
        if (per_sm < 1) per_sm = 1;
        int64_t ntiles = (p.R + p.TR - 1) / p.TR;
        int sms = device_info().sm_count;
        if (max_sms > 0 && max_sms < sms) sms = max_sms;
        int64_t grid = static_cast<int64_t>(sms) * per_sm;
        if (grid > ntiles) grid = ntiles;
        if (grid < 1) grid = 1;
        static const bool trace = std::getenv("KR_TRACE_PLAN") != nullptr;
        if (trace)
            std::fprintf(stderr, "[kr plan] %s R=%lld TR=%d threads=%d+32 rounds=%d stages=%d "
                         "mode=%d stage_bytes=%u smem=%zu grid=%lld per_sm=%d\n", name,
                         static_cast<long long>(p.R), p.TR, p.threads, p.rounds, p.stages, p.mode,
                         p.stage_bytes, smem, static_cast<long long>(grid), per_sm);
        kern<<<static_cast<unsigned>(grid), p.threads + 32, smem, st>>>(p, w, extra...);
        return check_launch(name);
    };
    return p.mode == kModeDirect ? go(kdirect) : go(kstaged);
}

}  // namespace kr

using namespace kr;

extern "C" int kr_horizon_static(int64_t R, int32_t N, int32_t static_h, int32_t* H,
                                 void* stream) {
    if (R < 0 || N < 1 || static_h < 1 || (R > 0 && !H)) return KR_EINVAL;
    if (R == 0) return KR_OK;
    int32_t h = static_h < N ? static_h : N;  // horizon.py:121-122
    int64_t blocks = (R + 255) / 256;
    if (blocks > 4096) blocks = 4096;
    k_horizon_static<<<static_cast<unsigned>(blocks), 256, 0, as_stream(stream)>>>(R, h, H);
    return check_launch("kr_horizon_static");
}

extern "C" int kr_horizon_confidence(const void* U, int dtype, int64_t R, int32_t K, int32_t N,
                                     double one_plus_t, int32_t min_horizon, int32_t* H,
                                     uint32_t* flags, void* stream) {
    if (R < 0 || K < 2 || N < 1 || min_horizon < 1 || (dtype != KR_F32 && dtype != KR_F64))
        return KR_EINVAL;
    if (R == 0) return KR_OK;
    if (!U || !H) return KR_EINVAL;
    const size_t es = dtype == KR_F64 ? 8 : 4;
    uint64_t rb = static_cast<uint64_t>(K) * N * es;
    if (N > (kStreamThreads - 32) * kMaxRounds) return KR_EINVAL;
    const void* bases[1] = {U};
    const float c1 = static_cast<float>(one_plus_t / static_cast<double>(K - 1));
    cudaStream_t st = as_stream(stream);
    auto go = [&](auto proto, auto kstaged, auto kdirect) {
        using W = decltype(proto);
        constexpr int VC = W::kVC;
        // two items per thread per tile: measured 80% -> 92% of the HBM peak
        // (K=6, N=50 fp32) from the amortised per-tile ring handshake
        StreamPlan p = make_plan(1, bases, &rb, R, N / VC, kMaxStages * sizeof(int),
                                 conf_max_threads<VC>() - 32, kernel_regs(kstaged), 2);
        const float m = static_cast<float>(K + 8) * 5.9604645e-8f;
        const double md = 1.7763568394002505e-15;  // 2^-49
        W w{K,       N,       p.TR,    min_horizon, p.rounds, one_plus_t,
            c1,      1.f + m, 1.f - m, one_plus_t / static_cast<double>(K - 1),
            1.0 + md, 1.0 - md, H,     flags,       nullptr,  {},
            {}};
        return launch_stream(kstaged, kdirect, p, w, st, "kr_horizon_confidence");
    };
    // columns per thread: vector loads need N % VC == 0 and a 16-byte aligned base
    const bool al = (reinterpret_cast<uintptr_t>(U) & 15u) == 0;
    int vc = !al || N % 2 ? 1 : (es == 4 && N % 4 == 0 ? 4 : 2);
    if (vc > 1 && N / vc > (conf_max_threads<2>() - 32) * kMaxRounds) vc = 1;
#define KR_CONF(TT, KK, VV)                                                                \
    return go(ConfWork<TT, KK, VV>{}, k_horizon_confidence<TT, KK, VV, true>,              \
              k_horizon_confidence<TT, KK, VV, false>)
#define KR_CONF_VC(TT, KK)                 \
    do {                                   \
        if (vc == 4) KR_CONF(TT, KK, 4);   \
        if (vc == 2) KR_CONF(TT, KK, 2);   \
        KR_CONF(TT, KK, 1);                \
    } while (0)
    if (dtype == KR_F64) {
        if (vc == 2) {
            if (K == 6) KR_CONF(double, 6, 2);
            KR_CONF(double, 0, 2);
        }
        if (K == 6) KR_CONF(double, 6, 1);
        KR_CONF(double, 0, 1);
    }
    if (K == 6) KR_CONF_VC(float, 6);
    KR_CONF_VC(float, 0);
#undef KR_CONF_VC
#undef KR_CONF
}

extern "C" int kr_horizon_sweep(const void* U, int dtype, int64_t R, int32_t K, int32_t N,
                                int32_t C, const int32_t* kind, const double* one_plus_t,
                                const int32_t* param, unsigned long long* sums, int32_t* H,
                                uint32_t* flags, void* stream) {
    if (R < 0 || K < 2 || N < 1 || C < 1 || C > kSweepMaxCfg || !kind || !one_plus_t || !param ||
        (dtype != KR_F32 && dtype != KR_F64))
        return KR_EINVAL;
    if (R == 0) return KR_OK;
    if (!U || !sums) return KR_EINVAL;
    if (N > (kStreamThreads - 32) * kMaxRounds) return KR_EINVAL;
    // configuration table: confidence slots first, ascending 1 + t (stable)
    SweepCfg cfg{};
    int order[kSweepMaxCfg];
    int Cc = 0;
    for (int c = 0; c < C; c++) {
        if (kind[c] != 0 && kind[c] != 1) return KR_EINVAL;
        if (kind[c] == 1) {
            if (!(one_plus_t[c] >= 1.0) || param[c] < 1) return KR_EINVAL;
            order[Cc++] = c;
        } else if (param[c] < 1) {
            return KR_EINVAL;
        }
    }
    for (int a = 1; a < Cc; a++)  // insertion sort (C <= 64)
        for (int b = a; b > 0 && one_plus_t[order[b - 1]] > one_plus_t[order[b]]; b--) {
            const int t = order[b];
            order[b] = order[b - 1];
            order[b - 1] = t;
        }
    int s = Cc;
    for (int c = 0; c < C; c++)
        if (kind[c] == 0) order[s++] = c;
    cfg.C = C;
    cfg.Cc = Cc;
    int P = 1;
    while (P <= Cc) P <<= 1;  // power of two > Cc: table entry P - 1 is +inf
    cfg.half = P / 2;
    // ratio bounds: c = (1 + t) / (K - 1) widened by the filter margin and
    // rounded outward in the storage type
    const bool f32 = dtype == KR_F32;
    const double mrg = f32 ? static_cast<double>(K + 8) * 5.9604644775390625e-8 : 1.7763568394002505e-15;
    for (int i = 0; i < kSweepPad; i++) {
        if (i < Cc) {
            const double c = one_plus_t[order[i]] / static_cast<double>(K - 1);
            if (f32) {
                cfg.rh[i] = std::nextafter(static_cast<float>(c * (1.0 + mrg)), INFINITY);
                cfg.rl[i] = std::nextafter(static_cast<float>(c * (1.0 - mrg)), 0.0f);
            } else {
                cfg.rh[i] = std::nextafter(c * (1.0 + mrg), INFINITY);
                cfg.rl[i] = std::nextafter(c * (1.0 - mrg), 0.0);
            }
        } else {
            cfg.rh[i] = cfg.rl[i] = INFINITY;
        }
    }
    // the filter runs for column sums in [sfmin, sfmax]: every ratio below
    // 2^100 / above 2^-100 of the sum is a normal number in both types
    cfg.sfmin = f32 ? 1e-30 : 1e-290;
    cfg.sfmax = f32 ? 1e30 : 1e290;
    if (!f32 && N < 2) cfg.sfmin = INFINITY;  // fp64 filter assumes the sequential mean order
    // bucket table over [2^floor(log2 rl[0]), 2^(floor(log2 rh[Cc-1]) + 1)):
    // 2^mbits buckets per binade
    cfg.lut_n = 1;  // default: one ambiguous bucket covering everything
    cfg.lut_lo = 0;
    cfg.lut_hi = f32 ? 0xFFFFFFFFull : ~uint64_t(0);  // above the largest ratio pattern
    cfg.lut_shift = f32 ? 31 : 63;
    cfg.lut[0] = 0xFFFF;
    if (Cc > 0 && std::isnormal(cfg.rl[0]) && std::isfinite(cfg.rh[Cc - 1]) &&
        (!f32 || (cfg.rl[0] > 1e-37 && cfg.rh[Cc - 1] < 1e37))) {
        int e_lo, e_hi;
        std::frexp(cfg.rl[0], &e_lo);       // rl[0] in [2^(e_lo-1), 2^e_lo)
        std::frexp(cfg.rh[Cc - 1], &e_hi);  // rh    in [2^(e_hi-1), 2^e_hi)
        const double lo = std::ldexp(1.0, e_lo - 1), hi = std::ldexp(1.0, e_hi);
        const int binades = e_hi - e_lo + 1;
        int mbits = 7;
        while (mbits > 0 && (binades << mbits) > kSweepLut) mbits--;
        if ((binades << mbits) <= kSweepLut && (f32 || binades < 2000)) {
            const int mant = f32 ? 23 : 52;
            cfg.lut_shift = mant - mbits;
            cfg.lut_n = binades << mbits;
            auto bits_of = [&](double x) -> uint64_t {
                if (f32) { const float f = static_cast<float>(x); uint32_t b; std::memcpy(&b, &f, 4); return b; }
                uint64_t b; std::memcpy(&b, &x, 8); return b;
            };
            auto val_of = [&](uint64_t b) -> double {
                if (f32) { const uint32_t b32 = static_cast<uint32_t>(b); float f; std::memcpy(&f, &b32, 4); return f; }
                double d; std::memcpy(&d, &b, 8); return d;
            };
            cfg.lut_lo = bits_of(lo);
            cfg.lut_hi = bits_of(hi);
            for (int bkt = 0; bkt < cfg.lut_n; bkt++) {
                const uint64_t b0 = cfg.lut_lo + (static_cast<uint64_t>(bkt) << cfg.lut_shift);
                const double x0 = val_of(b0);
                const double x1 = val_of(b0 + (uint64_t(1) << cfg.lut_shift) - 1);  // largest in bucket
                int a = 0, nb = 0;
                for (int i = 0; i < Cc; i++) {
                    a += cfg.rh[i] < x0;    // every ratio in the bucket is a definite trip
                    nb += cfg.rl[i] <= x1;  // some ratio in the bucket is not a definite non-trip
                }
                cfg.lut[bkt] = a == nb ? static_cast<uint16_t>(a) : uint16_t(0xFFFF);
            }
        }
    }
    for (int i = 0; i < C; i++) {
        const int c = order[i];
        cfg.orig[i] = c;
        cfg.hcap[i] = param[c] < N ? param[c] : N;  // horizon.py:121-122, 130-131
        if (i < Cc) {
            cfg.p[i] = one_plus_t[c];
            if (cfg.hcap[i] > cfg.maxcap) cfg.maxcap = cfg.hcap[i];
        }
    }
    const size_t es = dtype == KR_F64 ? 8 : 4;
    uint64_t rb = static_cast<uint64_t>(K) * N * es;
    const void* bases[1] = {U};
    cudaStream_t st = as_stream(stream);
    auto go = [&](auto proto, auto kstaged, auto kdirect) -> int {
        using W = decltype(proto);
        constexpr int VC = W::kVC;
        // a warp per robot (32 "items"): 11 consumer warps x 2 robots per tile,
        // two CTAs (24 warps) per SM -- the per-robot scan is instruction-heavy,
        // so warps, not bytes in flight, set the pace
        StreamPlan p = make_plan(1, bases, &rb, R, 32, 0, kSweepThreads - 32, kernel_regs(kstaged),
                                 2, static_cast<uint32_t>(sizeof(SweepTables)), 22);
        // per-CTA 32-bit sums: robots per CTA (grid >= SMs) x N < 2^32
        if ((R / device_info().sm_count + 1) * static_cast<int64_t>(N) >= (int64_t(1) << 32))
            return KR_EINVAL;
        W w{};
        w.K = K; w.N = N; w.TR = p.TR; w.C = C; w.Cc = Cc; w.maxcap = cfg.maxcap;
        w.half = cfg.half;
        w.cw = p.threads / 32;
        w.sfmin = static_cast<typename W::Elem>(cfg.sfmin);
        w.sfmax = static_cast<typename W::Elem>(cfg.sfmax);
        w.lut_n = cfg.lut_n; w.lut_shift = cfg.lut_shift; w.lut_lo = cfg.lut_lo; w.lut_hi = cfg.lut_hi;
        w.H = H; w.sums = sums; w.flags = flags; w.R = R;
        return launch_stream(kstaged, kdirect, p, w, st, "kr_horizon_sweep", 0, cfg);
    };
    // columns per lane: the fewest 32-lane chunks, then the most lanes busy
    const bool al = (reinterpret_cast<uintptr_t>(U) & 15u) == 0;
    int vc = 1;
    if (al && N % 2 == 0 && N > 32) vc = 2;
    if (al && es == 4 && N % 4 == 0 && N > 64) vc = 4;
#define KR_SWEEP(TT, KK, VV) \
    return go(SweepWork<TT, KK, VV>{}, k_horizon_sweep<TT, KK, VV, true>, k_horizon_sweep<TT, KK, VV, false>)
    if (dtype == KR_F64) {
        if (vc == 2) {
            if (K == 6) KR_SWEEP(double, 6, 2);
            KR_SWEEP(double, 0, 2);
        }
        KR_SWEEP(double, 0, 1);
    }
    if (vc == 4) {
        if (K == 6) KR_SWEEP(float, 6, 4);
        KR_SWEEP(float, 0, 4);
    }
    if (vc == 2) {
        if (K == 6) KR_SWEEP(float, 6, 2);
        KR_SWEEP(float, 0, 2);
    }
    KR_SWEEP(float, 0, 1);
#undef KR_SWEEP
}

template <typename T, bool SL>
static int launch_div(const StreamPlan& p, const DivWork<T, 0>& w0, cudaStream_t st, int max_sms) {
    auto with = [&](auto proto) {
        decltype(proto) w{w0.S, w0.Lp, w0.Lc, w0.D, w0.TR, w0.rounds, w0.has_off, w0.has_lp,
                          w0.has_lc, w0.thr, w0.H, w0.cos, w0.thr_f, w0.margin, nullptr, nullptr,
                          {}, {}, {}};
        return w;
    };
    switch (w0.D) {
        case 7:
            return launch_stream(k_horizon_divergence<T, 7, true, SL>,
                                 k_horizon_divergence<T, 7, false, SL>, p,
                                 with(DivWork<T, 7, SL>{}), st, "kr_horizon_divergence", max_sms);
        case 32:
            return launch_stream(k_horizon_divergence<T, 32, true, SL>,
                                 k_horizon_divergence<T, 32, false, SL>, p,
                                 with(DivWork<T, 32, SL>{}), st, "kr_horizon_divergence", max_sms);
        default:
            return launch_stream(k_horizon_divergence<T, 0, true, SL>,
                                 k_horizon_divergence<T, 0, false, SL>, p,
                                 with(DivWork<T, 0, SL>{}), st, "kr_horizon_divergence", max_sms);
    }
}

template <typename T, bool SL>
static int div_regs(int D) {
    return D == 7 ? kernel_regs(k_horizon_divergence<T, 7, true, SL>)
                  : (D == 32 ? kernel_regs(k_horizon_divergence<T, 32, true, SL>)
                             : kernel_regs(k_horizon_divergence<T, 0, true, SL>));
}

extern "C" int kr_horizon_divergence(const void* prev, const void* cand, int dtype, int64_t R,
                                     int32_t S, int32_t Lp, int32_t Lc, int32_t D,
                                     const int32_t* offset, const int32_t* len_prev,
                                     const int32_t* len_cand, double thr, int32_t* H, double* cos,
                                     int32_t max_sms, void* stream) {
    if (R < 0 || S < 1 || Lp < 0 || Lc < 0 || D < 0 || (dtype != KR_F32 && dtype != KR_F64))
        return KR_EINVAL;
    if (!(thr > 0.0 && thr <= 1.0)) return KR_EINVAL;  // workload.py:483-484
    if (R == 0) return KR_OK;
    const size_t es = dtype == KR_F64 ? 8 : 4;
    uint64_t rb[2] = {static_cast<uint64_t>(Lp) * D * es, static_cast<uint64_t>(S) * Lc * D * es};
    if (!H || (rb[0] && !prev) || (rb[1] && !cand)) return KR_EINVAL;
    if (Lp == 0 || Lc == 0) {  // empty trajectories: every horizon is 0
        cudaStream_t st = as_stream(stream);
        KR_CUDA_TRY(cudaMemsetAsync(H, 0, R * sizeof(int32_t), st));
        if (cos && Lc > 0)
            KR_CUDA_TRY(cudaMemsetAsync(cos, 0xFF, R * S * Lc * sizeof(double), st));
        return KR_OK;
    }
    // S > 1: a thread per (robot, action) loops over the samples
    const bool sl = S > 1;
    const int64_t items = sl ? Lc : static_cast<int64_t>(S) * Lc;
    if (items > static_cast<int64_t>(kStreamThreads) * kMaxRounds) return KR_EINVAL;
    // segments: action rows, then the per-robot metadata that travels with them
    const void* bases[5] = {prev, cand, offset, len_prev, len_cand};
    uint64_t rbs[5] = {rb[0], rb[1], offset ? 4u : 0u, len_prev ? 4u : 0u, len_cand ? 4u : 0u};
    const int nseg = 5;
    const int maxt = D == 7 ? kStreamThreads : 256;  // only D = 7 has a small-D kernel
    if (items > static_cast<int64_t>(maxt - 32) * kMaxRounds) return KR_EINVAL;
    const bool f64 = dtype == KR_F64;
    const int regs = f64 ? (sl ? div_regs<double, true>(D) : div_regs<double, false>(D))
                         : (sl ? div_regs<float, true>(D) : div_regs<float, false>(D));
    StreamPlan p = make_plan(nseg, bases, rbs, R, static_cast<int>(items),
                             2 * kMaxStages * sizeof(int), maxt - 32, regs);
    cudaStream_t st = as_stream(stream);
    const float thr_f = static_cast<float>(thr);
    const float margin = cos_filter_margin(D);
    if (f64) {
        DivWork<double, 0> w{S, Lp, Lc, D, p.TR, p.rounds, offset != nullptr, len_prev != nullptr,
                             len_cand != nullptr, thr, H, cos, thr_f, margin, nullptr, nullptr,
                             {}, {}, {}};
        return sl ? launch_div<double, true>(p, w, st, max_sms)
                  : launch_div<double, false>(p, w, st, max_sms);
    }
    DivWork<float, 0> w{S, Lp, Lc, D, p.TR, p.rounds, offset != nullptr, len_prev != nullptr,
                        len_cand != nullptr, thr, H, cos, thr_f, margin, nullptr, nullptr,
                        {}, {}, {}};
    return sl ? launch_div<float, true>(p, w, st, max_sms) : launch_div<float, false>(p, w, st, max_sms);
}
