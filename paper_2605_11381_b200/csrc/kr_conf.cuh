// kr_conf.cuh -- confidence-threshold policy (horizon.py:108-132) device code,
// shared by k_horizon_confidence (kr_horizon.cu) and k_horizon_sweep
// (kr_sweep.cu).
#pragma once

#include <climits>

#include "kr_common.cuh"
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
        // an exact zero mean: the reference's threshold (1 + t) * 0.0 is 0 for
        // finite 1 + t, so any f > 0 trips (NaN for t = inf / NaN: never) --
        // decided here directly, since c1 overflows to inf for thresholds
        // beyond FLT_MAX and thr = 0 * inf would be NaN
        const bool zero_mean = sf == T(0);
        und = !(fin == T(0) || zero_mean || (in_range && (hi || lo)));
        return zero_mean ? (fin > T(0) && isfinite(opt)) : hi;
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

}  // namespace kr
