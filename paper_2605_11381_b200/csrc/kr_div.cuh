// kr_div.cuh -- the divergence-horizon kernel family (workload.py:461-496):
// per-timestep cosine divergence between each new chunk (S samples) and the
// unexecuted overlap of the previous chunk, reduced to the longest prefix that
// stays at or above the similarity threshold.  Templated on ORD, the OpenBLAS
// core whose ddot order the exact fp64 cosines follow (kDotSkylakeX /
// kDotHaswell, see kr_common.cuh); each order is instantiated in its own
// translation unit (kr_div_skx.cu, kr_div_hsw.cu) and selected per launch by
// kr_horizon_divergence from the process-wide kr_set_dot_order setting.
#pragma once
#include <climits>
#include <cmath>
#include <cstring>
#include <type_traits>
#include <cstdio>
#include <cstdlib>

#include "kr_common.cuh"
#include "kr_host.cuh"
#include "kr_stream.cuh"
#include "kr_plan.cuh"

namespace kr {

#ifndef KR_SHARED_STAGES
#define KR_SHARED_STAGES 3
#endif
constexpr int kSharedStages = KR_SHARED_STAGES;  // ring depth when the horizon kernel shares the GPU

// ---------------------------------------------------------------------------
// Divergence horizon (workload.py:461-496), S-sample ensembles, ragged rows
// ---------------------------------------------------------------------------
// SL ("samples looped", S > 1): one thread per (robot, action) scores all S
// samples against the reference row it loads once (kept in registers for
// small D); the robot's horizon is the first action where ANY sample falls
// below the threshold, so one first-trip reduction per action suffices.
template <typename T, int DC, bool SL = false, int ORD = kDotSkylakeX>
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
                    const double c = cosine_ord_fixed<DC, ORD>(a, b);
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
                        c = cosine_ord_fixed<DC, ORD>(a, b);
                    else
                        c = cosine_ord<ORD>(a, b, D_);
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
                            c = cosine_ord_fixed<DC, ORD>(a, b);
                        else
                            c = cosine_ord<ORD>(a, b, D_);
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

template <typename T, int DC, bool kStaged, bool SL = false, int ORD = kDotSkylakeX>
__global__ void __launch_bounds__(div_max_threads<DC>()) k_horizon_divergence(StreamPlan p,
                                                                             DivWork<T, DC, SL, ORD> w) {
    extern __shared__ __align__(128) unsigned char smem[];
    w.first = reinterpret_cast<int*>(smem + stream_aux_offset());
    w.lim = w.first + kMaxStages * w.TR;
    for (int i = threadIdx.x; i < kMaxStages * w.TR; i += blockDim.x) w.first[i] = INT_MAX;
    w.setup(p.threads);
    __syncthreads();
    stream_run<kStaged>(p, smem, w);
}

// Arguments of one kr_horizon_divergence call (validated, non-empty).
struct DivArgs {
    const void* prev;
    const void* cand;
    int dtype;
    int64_t R;
    int32_t S, Lp, Lc, D;
    const int32_t* offset;
    const int32_t* len_prev;
    const int32_t* len_cand;
    double thr;
    int32_t* H;
    double* cos;
    int32_t max_sms;
    void* stream;
};

template <typename T, bool SL, int ORD>
int launch_div(const StreamPlan& p, const DivWork<T, 0>& w0, cudaStream_t st, int max_sms) {
    auto with = [&](auto proto) {
        decltype(proto) w{w0.S, w0.Lp, w0.Lc, w0.D, w0.TR, w0.rounds, w0.has_off, w0.has_lp,
                          w0.has_lc, w0.thr, w0.H, w0.cos, w0.thr_f, w0.margin, nullptr, nullptr,
                          {}, {}, {}};
        return w;
    };
    if constexpr (SL) {  // ensembles: D = 7 specialised, every other D generic
        if (w0.D == 7)
            return launch_stream(k_horizon_divergence<T, 7, true, SL, ORD>,
                                 k_horizon_divergence<T, 7, false, SL, ORD>, p,
                                 with(DivWork<T, 7, SL, ORD>{}), st, "kr_horizon_divergence", max_sms);
        return launch_stream(k_horizon_divergence<T, 0, true, SL, ORD>,
                             k_horizon_divergence<T, 0, false, SL, ORD>, p,
                             with(DivWork<T, 0, SL, ORD>{}), st, "kr_horizon_divergence", max_sms);
    }
    switch (w0.D) {
        case 7:
            return launch_stream(k_horizon_divergence<T, 7, true, SL, ORD>,
                                 k_horizon_divergence<T, 7, false, SL, ORD>, p,
                                 with(DivWork<T, 7, SL, ORD>{}), st, "kr_horizon_divergence", max_sms);
        case 32:
            return launch_stream(k_horizon_divergence<T, 32, true, SL, ORD>,
                                 k_horizon_divergence<T, 32, false, SL, ORD>, p,
                                 with(DivWork<T, 32, SL, ORD>{}), st, "kr_horizon_divergence", max_sms);
        default:
            return launch_stream(k_horizon_divergence<T, 0, true, SL, ORD>,
                                 k_horizon_divergence<T, 0, false, SL, ORD>, p,
                                 with(DivWork<T, 0, SL, ORD>{}), st, "kr_horizon_divergence", max_sms);
    }
}

template <typename T, bool SL, int ORD>
int div_regs(int D) {
    if constexpr (SL)
        return D == 7 ? kernel_regs(k_horizon_divergence<T, 7, true, SL, ORD>)
                      : kernel_regs(k_horizon_divergence<T, 0, true, SL, ORD>);
    return D == 7 ? kernel_regs(k_horizon_divergence<T, 7, true, SL, ORD>)
                  : (D == 32 ? kernel_regs(k_horizon_divergence<T, 32, true, SL, ORD>)
                             : kernel_regs(k_horizon_divergence<T, 0, true, SL, ORD>));
}

template <int ORD>
int div_run(const DivArgs& a) {
    const void* prev = a.prev;
    const void* cand = a.cand;
    const int dtype = a.dtype;
    const int64_t R = a.R;
    const int32_t S = a.S, Lp = a.Lp, Lc = a.Lc, D = a.D;
    const int32_t* offset = a.offset;
    const int32_t* len_prev = a.len_prev;
    const int32_t* len_cand = a.len_cand;
    const double thr = a.thr;
    int32_t* H = a.H;
    double* cos = a.cos;
    const int32_t max_sms = a.max_sms;
    void* stream = a.stream;
    const size_t es = dtype == KR_F64 ? 8 : 4;
    uint64_t rb[2] = {static_cast<uint64_t>(Lp) * D * es, static_cast<uint64_t>(S) * Lc * D * es};
    // S > 1: a thread per (robot, action) loops over the samples
    const bool sl = S > 1 && dtype == KR_F32;  // fp64 ensembles take the per-sample items
    const int64_t items = sl ? Lc : static_cast<int64_t>(S) * Lc;
    if (items > static_cast<int64_t>(kStreamThreads) * kMaxRounds) return KR_EINVAL;
    // segments: action rows, then the per-robot metadata that travels with them
    const void* bases[5] = {prev, cand, offset, len_prev, len_cand};
    uint64_t rbs[5] = {rb[0], rb[1], offset ? 4u : 0u, len_prev ? 4u : 0u, len_cand ? 4u : 0u};
    const int nseg = 5;
    const int maxt = D == 7 ? kStreamThreads : 256;  // only D = 7 has a small-D kernel
    if (items > static_cast<int64_t>(maxt - 32) * kMaxRounds) return KR_EINVAL;
    const bool f64 = dtype == KR_F64;
    const int regs = f64 ? div_regs<double, false, ORD>(D)
                         : (sl ? div_regs<float, true, ORD>(D) : div_regs<float, false, ORD>(D));
    // Sharing the GPU with the round's admission (max_sms > 0): a ring of at
    // most 3 stages, so the planner takes a wider tile with fewer threads and
    // the side stream's kernels co-reside on the horizon SMs too (measured:
    // side stream 0.40 -> 0.21 ms, round -2%).
    StreamPlan p = make_plan(nseg, bases, rbs, R, static_cast<int>(items),
                             2 * kMaxStages * sizeof(int), maxt - 32, regs, 1, 256, 0,
                             max_sms > 0 ? kSharedStages : kMaxStages);
    cudaStream_t st = as_stream(stream);
    const float thr_f = static_cast<float>(thr);
    const float margin = cos_filter_margin(D);
    if (f64) {
        DivWork<double, 0> w{S, Lp, Lc, D, p.TR, p.rounds, offset != nullptr, len_prev != nullptr,
                             len_cand != nullptr, thr, H, cos, thr_f, margin, nullptr, nullptr,
                             {}, {}, {}};
        return launch_div<double, false, ORD>(p, w, st, max_sms);
    }
    DivWork<float, 0> w{S, Lp, Lc, D, p.TR, p.rounds, offset != nullptr, len_prev != nullptr,
                        len_cand != nullptr, thr, H, cos, thr_f, margin, nullptr, nullptr,
                        {}, {}, {}};
    return sl ? launch_div<float, true, ORD>(p, w, st, max_sms) : launch_div<float, false, ORD>(p, w, st, max_sms);
}

int div_run_skx(const DivArgs& a);  // kr_div_skx.cu
int div_run_hsw(const DivArgs& a);  // kr_div_hsw.cu

}  // namespace kr
