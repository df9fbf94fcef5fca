// kr_common.cuh -- device-side building blocks shared by every kernel of the
// Kairos decision core: bit-exact fp64 numerics that reproduce the reference's
// numpy / OpenBLAS evaluation order, integer-microsecond time arithmetic, the
// wait ledger, the packed composite sort key, and the sm_100a PTX wrappers for
// TMA bulk copies and mbarriers.
//
// Everything here is compiled with -fmad=false and uses explicit _rn
// intrinsics, so no fp64 operation is contracted or reassociated: the fused
// multiply-adds below exist exactly where OpenBLAS 0.3.30 (SkylakeX kernel)
// fuses (see oracle/kairos_oracle.c for the matching CPU restatement).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/kairos_b200.h"

namespace kr {

constexpr int kMaxThreads = 256;

// ---------------------------------------------------------------------------
// PTX: shared-memory addresses, mbarriers, 1-D TMA bulk copies
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(
                     smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "KR_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra KR_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// Programmatic dependent launch: wait until the same-stream predecessor grid
// has completed and its memory is visible (a no-op for a plain launch).
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Global -> shared bulk copy through the TMA engine; completion is signalled
// as transaction bytes on `bar`.  dst, src and bytes must be 16-byte aligned.
// The evict-first L2 policy keeps the one-pass action-chunk stream from
// displacing the (re-read) fleet state and sort keys.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
// Generic-proxy accesses to shared memory must be ordered before a
// subsequent async-proxy (TMA) write to the same buffer.
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---------------------------------------------------------------------------
// fp64 arithmetic with explicit rounding (never contracted)
// ---------------------------------------------------------------------------
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dfma(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double dsqrt(double a) { return __dsqrt_rn(a); }

template <typename T>
__device__ __forceinline__ double to_f64(T v) { return static_cast<double>(v); }

// numpy DOUBLE_pairwise_sum (numpy 2.3, loops_utils.h.src): used by
// `u[:-1].mean(axis=0)` when N == 1 (horizon.py:125).  The
// recursion splits at a multiple of 8 until blocks of <= 128, which are
// reduced with 8 accumulators.
template <class F>
__device__ double np_pairwise_block(F a, int64_t lo, int64_t n) {
    if (n < 8) {
        double res = 0.0;
        for (int64_t i = 0; i < n; i++) res = dadd(res, a(lo + i));
        return res;
    }
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; j++) r[j] = a(lo + j);
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8) {
#pragma unroll
        for (int j = 0; j < 8; j++) r[j] = dadd(r[j], a(lo + i + j));
    }
    double res = dadd(dadd(dadd(r[0], r[1]), dadd(r[2], r[3])),
                      dadd(dadd(r[4], r[5]), dadd(r[6], r[7])));
    for (; i < n; i++) res = dadd(res, a(lo + i));
    return res;
}

template <class F>
__device__ double np_pairwise_sum(F a, int64_t lo, int64_t n) {
    if (n <= 128) return np_pairwise_block(a, lo, n);
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return dadd(np_pairwise_sum(a, lo, n2), np_pairwise_sum(a, lo + n2, n - n2));
}

// OpenBLAS 0.3.30 ddot, contiguous, SkylakeX micro-kernel order
// (kernel/x86_64/ddot.c + ddot_microk_skylakex-2.c): n & -16 elements through
// 4x8-lane FMA accumulators over 32-blocks, folded to 4x4 lanes, 4x4-lane FMA
// over remaining 16-blocks, lane chain, (a0+a2)+(a1+a3); scalar FMA tail.
template <class FX, class FY>
__device__ __forceinline__ double ddot_skx(FX x, FY y, int n) {
    int n1 = n & -16, n32 = n1 & ~31, i = 0;
    double dot = 0.0;
    if (n1) {
        double acc[32];
#pragma unroll
        for (int e = 0; e < 32; e++) acc[e] = 0.0;
        for (; i < n32; i += 32) {
#pragma unroll
            for (int e = 0; e < 32; e++) acc[e] = dfma(x(i + e), y(i + e), acc[e]);
        }
        double a4[16];
#pragma unroll
        for (int j = 0; j < 4; j++)
#pragma unroll
            for (int l = 0; l < 4; l++) a4[4 * j + l] = dadd(acc[8 * j + l], acc[8 * j + l + 4]);
        for (; i < n1; i += 16) {
#pragma unroll
            for (int e = 0; e < 16; e++) a4[e] = dfma(x(i + e), y(i + e), a4[e]);
        }
        double a[4];
#pragma unroll
        for (int l = 0; l < 4; l++) a[l] = dadd(dadd(dadd(a4[l], a4[4 + l]), a4[8 + l]), a4[12 + l]);
        dot = dadd(dadd(a[0], a[2]), dadd(a[1], a[3]));
    }
    for (; i < n; i++) dot = dfma(y(i), x(i), dot);
    return dot;
}

// workload.py:461-468 `_cosine(a, b)` with a = candidate action, b = reference
// action.  For D < 16 the three OpenBLAS dots are plain FMA chains, evaluated
// in one pass so each element is loaded once.
template <typename T>
__device__ __forceinline__ double cosine_skx(const T* a, const T* b, int D) {
    double xx, yy, xy;
    if (D < 16) {
        xx = 0.0; yy = 0.0; xy = 0.0;
        for (int i = 0; i < D; i++) {
            double x = to_f64(a[i]), y = to_f64(b[i]);
            xx = dfma(x, x, xx);
            yy = dfma(y, y, yy);
            xy = dfma(y, x, xy);
        }
    } else {
        auto fa = [a](int i) { return to_f64(a[i]); };
        auto fb = [b](int i) { return to_f64(b[i]); };
        xx = ddot_skx(fa, fa, D);
        yy = ddot_skx(fb, fb, D);
        xy = ddot_skx(fa, fb, D);
    }
    double na = dsqrt(xx), nb = dsqrt(yy);
    if (na == 0.0 && nb == 0.0) return 1.0;
    if (na == 0.0 || nb == 0.0) return 0.0;
    return ddiv(xy, dmul(na, nb));
}

// Compile-time-D variant for the hot shapes: fully unrolled, operands held in
// registers after one pass over shared memory.
template <int DC, typename T>
__device__ __forceinline__ double cosine_skx_fixed(const T* a, const T* b) {
    double x[DC], y[DC];
#pragma unroll
    for (int i = 0; i < DC; i++) {
        x[i] = to_f64(a[i]);
        y[i] = to_f64(b[i]);
    }
    double xx, yy, xy;
    if constexpr (DC < 16) {
        xx = 0.0; yy = 0.0; xy = 0.0;
#pragma unroll
        for (int i = 0; i < DC; i++) {
            xx = dfma(x[i], x[i], xx);
            yy = dfma(y[i], y[i], yy);
            xy = dfma(y[i], x[i], xy);
        }
    } else {
        auto fx = [&](int i) { return x[i]; };
        auto fy = [&](int i) { return y[i]; };
        xx = ddot_skx(fx, fx, DC);
        yy = ddot_skx(fy, fy, DC);
        xy = ddot_skx(fx, fy, DC);
    }
    double na = dsqrt(xx), nb = dsqrt(yy);
    if (na == 0.0 && nb == 0.0) return 1.0;
    if (na == 0.0 || nb == 0.0) return 0.0;
    return ddiv(xy, dmul(na, nb));
}

// The same library's Haswell core (selected on Haswell and Zen hosts; read
// from the installed libscipy_openblas' ddot kernel for that core and pinned
// against numpy under OPENBLAS_CORETYPE=Haswell): n & -16 elements through
// 4x4-lane FMA accumulators over 16-blocks, each folding its lanes (m, m+2),
// then (h0+h1)+(h2+h3) per lane and r0+r1; the tail is an unfused
// `dot += y * x` (D < 16: only the tail).
template <class FX, class FY>
__device__ __forceinline__ double ddot_hsw(FX x, FY y, int n) {
    int n1 = n & -16, i = 0;
    double dot = 0.0;
    if (n1) {
        double acc[16];
#pragma unroll
        for (int e = 0; e < 16; e++) acc[e] = 0.0;
        for (; i < n1; i += 16) {
#pragma unroll
            for (int e = 0; e < 16; e++) acc[e] = dfma(x(i + e), y(i + e), acc[e]);
        }
        double r[2];
#pragma unroll
        for (int m = 0; m < 2; m++) {
            double h[4];
#pragma unroll
            for (int j = 0; j < 4; j++) h[j] = dadd(acc[4 * j + m], acc[4 * j + m + 2]);
            r[m] = dadd(dadd(h[0], h[1]), dadd(h[2], h[3]));
        }
        dot = dadd(r[0], r[1]);
    }
    for (; i < n; i++) dot = dadd(dot, dmul(y(i), x(i)));
    return dot;
}

// Which OpenBLAS core's ddot order the exact cosines follow (a kernel
// template parameter; the host picks it from kr_set_dot_order).
enum : int { kDotSkylakeX = 0, kDotHaswell = 1 };

__device__ __forceinline__ double cos_from_dots(double xx, double yy, double xy) {
    double na = dsqrt(xx), nb = dsqrt(yy);
    if (na == 0.0 && nb == 0.0) return 1.0;
    if (na == 0.0 || nb == 0.0) return 0.0;
    return ddiv(xy, dmul(na, nb));
}

// `_cosine` in the given core's order
template <int ORD, typename T>
__device__ __forceinline__ double cosine_ord(const T* a, const T* b, int D) {
    if constexpr (ORD == kDotSkylakeX) {
        return cosine_skx(a, b, D);
    } else {
        if (D < 16) {  // only the unfused tail: one pass, three chains
            double xx = 0.0, yy = 0.0, xy = 0.0;
            for (int i = 0; i < D; i++) {
                const double x = to_f64(a[i]), y = to_f64(b[i]);
                xx = dadd(xx, dmul(x, x));
                yy = dadd(yy, dmul(y, y));
                xy = dadd(xy, dmul(y, x));
            }
            return cos_from_dots(xx, yy, xy);
        }
        auto fa = [a](int i) { return to_f64(a[i]); };
        auto fb = [b](int i) { return to_f64(b[i]); };
        return cos_from_dots(ddot_hsw(fa, fa, D), ddot_hsw(fb, fb, D), ddot_hsw(fa, fb, D));
    }
}

template <int DC, int ORD, typename T>
__device__ __forceinline__ double cosine_ord_fixed(const T* a, const T* b) {
    if constexpr (ORD == kDotSkylakeX) {
        return cosine_skx_fixed<DC>(a, b);
    } else if constexpr (DC < 16) {  // only the unfused tail: one pass, three chains
        double xx = 0.0, yy = 0.0, xy = 0.0;
#pragma unroll
        for (int i = 0; i < DC; i++) {
            const double x = to_f64(a[i]), y = to_f64(b[i]);
            xx = dadd(xx, dmul(x, x));
            yy = dadd(yy, dmul(y, y));
            xy = dadd(xy, dmul(y, x));
        }
        return cos_from_dots(xx, yy, xy);
    } else {
        double x[DC], y[DC];
#pragma unroll
        for (int i = 0; i < DC; i++) {
            x[i] = to_f64(a[i]);
            y[i] = to_f64(b[i]);
        }
        auto fx = [&](int i) { return x[i]; };
        auto fy = [&](int i) { return y[i]; };
        return cos_from_dots(ddot_hsw(fx, fx, DC), ddot_hsw(fy, fy, DC), ddot_hsw(fx, fy, DC));
    }
}

// ---------------------------------------------------------------------------
// Exact fp32 pre-decision ("filter") for the cosine threshold test
// ---------------------------------------------------------------------------
// The reference decides `cos < thr` on an fp64 cosine.  For fp32-representable
// inputs an fp32 evaluation of the same cosine is within a proven bound of the
// exact value: every dot is off by at most gamma_D = D*2^-24 relative to
// sum|x_i*y_i| <= |x||y| (Cauchy-Schwarz), rsqrt.approx by 2^-22.9, and the
// two products by 1/2 ulp each, so |c32 - c| <= 2*gamma_D + 2^-21; the fp64
// result differs from c by < 2^-48.  Whenever |c32 - thr| exceeds
// margin = (2D + 24) * 2^-24 + 2^-20 the decision is therefore already known;
// only the rare near-threshold actions (and zero / extreme-range vectors) fall
// back to the bit-exact fp64 path.  Decisions are identical by construction.
__host__ __device__ inline float cos_filter_margin(int D) {
    return static_cast<float>((2.0 * D + 24.0) * 5.9604644775390625e-8 + 9.5367431640625e-7);
}

// Returns 1 (cos >= thr), 0 (cos < thr) or -1 (undecided: use the exact path).
// The bound holds for any summation order, so rows whose length is a multiple
// of 32 words are read starting at a lane-rotated element: lanes scoring
// consecutive rows (all starting at bank 0) then hit 32 distinct banks.
__device__ __forceinline__ float rsqrt_approx_ftz(float x) {
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
// c = xy / sqrt(xx * yy) with one MUFU: the range guard keeps xx * yy a normal
// float, and rsqrt.approx's 2^-22.9 relative error is inside the margin.
__device__ __forceinline__ int cos_filter_decide(float xx, float yy, float xy, float thr_f,
                                                 float margin) {
    if (!(xx >= 1e-18f && yy >= 1e-18f && xx <= 1e18f && yy <= 1e18f)) return -1;
    const float c = __fmul_rn(xy, rsqrt_approx_ftz(__fmul_rn(xx, yy)));
    const float d = __fsub_rn(c, thr_f);
    if (d > margin) return 1;
    if (d < -margin) return 0;
    return -1;
}

template <int DC, typename T>
__device__ __forceinline__ int cos_filter_fixed(const T* a, const T* b, float thr_f, float margin) {
    float xx = 0.f, yy = 0.f, xy = 0.f;
    if constexpr (DC % 32 == 0) {
        const int rot = threadIdx.x & 31;
#pragma unroll
        for (int e = 0; e < DC; e++) {
            const int i = (e + rot) % DC;
            const float x = static_cast<float>(a[i]), y = static_cast<float>(b[i]);
            xx = __fmaf_rn(x, x, xx);
            yy = __fmaf_rn(y, y, yy);
            xy = __fmaf_rn(x, y, xy);
        }
    } else {
#pragma unroll
        for (int i = 0; i < DC; i++) {
            const float x = static_cast<float>(a[i]), y = static_cast<float>(b[i]);
            xx = __fmaf_rn(x, x, xx);
            yy = __fmaf_rn(y, y, yy);
            xy = __fmaf_rn(x, y, xy);
        }
    }
    return cos_filter_decide(xx, yy, xy, thr_f, margin);
}
template <typename T>
__device__ __forceinline__ int cos_filter(const T* a, const T* b, int D, float thr_f, float margin) {
    float xx = 0.f, yy = 0.f, xy = 0.f;
    const int rot = (D % 32 == 0) ? (threadIdx.x & 31) : 0;
    int i = rot;
    for (int e = 0; e < D; e++) {
        const float x = static_cast<float>(a[i]), y = static_cast<float>(b[i]);
        xx = __fmaf_rn(x, x, xx);
        yy = __fmaf_rn(y, y, yy);
        xy = __fmaf_rn(x, y, xy);
        if (++i == D) i = 0;
    }
    return cos_filter_decide(xx, yy, xy, thr_f, margin);
}

// Magic-number unsigned division for n < 2^31 (loop-invariant divisors).
struct FastDiv {
    uint32_t d, m, s;
};
__host__ inline FastDiv make_fastdiv(uint32_t d) {
    uint32_t s = 0;
    while ((uint64_t(1) << s) < d) s++;
    uint64_t m = ((uint64_t(1) << 32) * ((uint64_t(1) << s) - d)) / d + 1;
    return FastDiv{d, static_cast<uint32_t>(m), s};
}
__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv& f) {
    return (__umulhi(n, f.m) + n) >> f.s;
}

// ---------------------------------------------------------------------------
// Integer-microsecond time (core.py:24-47)
// ---------------------------------------------------------------------------
// us_from_actions(count, hz_num/hz_den) = floor(count*1e6*den/num + 1/2)
//   = (2*count*1e6*den + num) div (2*num).
__device__ __forceinline__ int64_t us_from_actions(int64_t count, int64_t hz_num, int64_t hz_den,
                                                   uint32_t* flag_bits) {
    if (count < 0) {
        *flag_bits |= KR_FLAG_TIME_RANGE;
        return 0;
    }
    if (hz_den == 1 && count < (int64_t(1) << 40) && hz_num < (int64_t(1) << 40)) {
        int64_t X = count * 1000000;
        return (2 * X + hz_num) / (2 * hz_num);
    }
    unsigned __int128 X = (unsigned __int128)count * 1000000u * (unsigned __int128)hz_den;
    unsigned __int128 Y = (unsigned __int128)hz_num;
    unsigned __int128 q = (2 * X + Y) / (2 * Y);
    if (q > (unsigned __int128)INT64_MAX) *flag_bits |= KR_FLAG_TIME_RANGE;
    return (int64_t)q;
}

// ---------------------------------------------------------------------------
// Wait ledger (waiting.py:69-93), wait ratio (waiting.py:62-66, 96-100),
// bucket (scheduler.py:79-88)
// ---------------------------------------------------------------------------
__device__ __forceinline__ void l2_prefetch(const void* p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

struct Slot {
    int64_t gs, ge, es, ee;
};
__device__ __forceinline__ Slot load_slot(const int64_t* slots, int64_t j) {
    const longlong2* p = reinterpret_cast<const longlong2*>(slots + 4 * j);
    longlong2 a = __ldg(p), b = __ldg(p + 1);
    return Slot{a.x, a.y, b.x, b.y};
}

// Per round j < n_exec: gen-dominated (|G_j| >= |E_j|) rounds accrue
// max(0, G_{j+1}.start - G_j.end) once G_{j+1} has started (n_gen > j+1, the
// successor may still be in flight); exec-dominated rounds accrue
// max(0, E_{j+1}.start - E_j.end) once E_{j+1} exists; the last round none.
__device__ __forceinline__ int64_t total_wait(const int64_t* slots, int32_t n_exec,
                                              int32_t n_gen) {
    int64_t total = 0;
    if (n_exec <= 0) return 0;
    Slot cur = load_slot(slots, 0);
    for (int32_t j = 0; j < n_exec; j++) {
        bool has_next = (j + 1 < n_exec) || (n_gen > j + 1);
        Slot nxt = has_next ? load_slot(slots, j + 1) : Slot{0, 0, 0, 0};
        if (cur.ge - cur.gs >= cur.ee - cur.es) {
            if (n_gen > j + 1) {
                int64_t w = nxt.gs - cur.ge;
                total += w > 0 ? w : 0;
            }
        } else if (j + 1 < n_exec) {
            int64_t w = nxt.es - cur.ee;
            total += w > 0 ? w : 0;
        }
        cur = nxt;
    }
    return total;
}

// Round j's recorded wait given its successor slot (only the successor's
// generation / execution start is read), the per-round body of total_wait.
__device__ __forceinline__ int64_t round_wait(const Slot& cur, int64_t nxt_gs, int64_t nxt_es,
                                              int32_t j, int32_t n_exec, int32_t n_gen) {
    int64_t w = 0;
    if (cur.ge - cur.gs >= cur.ee - cur.es) {
        if (n_gen > j + 1) w = nxt_gs - cur.ge;
    } else if (j + 1 < n_exec) {
        w = nxt_es - cur.ee;
    }
    return w > 0 ? w : 0;
}

// total_wait plus the last execution's length, with the first four slots
// loaded up front (independent loads: one memory latency for a history of up
// to four slots instead of one per round); longer histories continue slot by
// slot.  Same per-round arithmetic as total_wait.
__device__ __forceinline__ void history_walk(const int64_t* slots, int32_t n_exec, int32_t n_gen,
                                             int64_t& total, int64_t& last) {
    total = 0;
    last = 0;
    if (n_exec <= 0) return;
    const int32_t ext = n_gen > n_exec ? n_gen : n_exec;
    const Slot z{0, 0, 0, 0};
    const Slot s0 = load_slot(slots, 0);
    const Slot s1 = ext > 1 ? load_slot(slots, 1) : z;
    const Slot s2 = ext > 2 ? load_slot(slots, 2) : z;
    const Slot s3 = ext > 3 ? load_slot(slots, 3) : z;
    total = round_wait(s0, s1.gs, s1.es, 0, n_exec, n_gen);
    if (n_exec > 1) total += round_wait(s1, s2.gs, s2.es, 1, n_exec, n_gen);
    if (n_exec > 2) total += round_wait(s2, s3.gs, s3.es, 2, n_exec, n_gen);
    // by value (a reference to one of the four would put them in local memory)
    last = n_exec == 1 ? s0.ee - s0.es : n_exec == 2 ? s1.ee - s1.es : n_exec == 3 ? s2.ee - s2.es
                                                                                  : s3.ee - s3.es;
    if (n_exec > 3) {  // rounds 3 .. n_exec-1
        Slot cur = s3;
        for (int32_t j = 3; j < n_exec; j++) {
            const Slot nxt = j + 1 < ext ? load_slot(slots, j + 1) : z;
            total += round_wait(cur, nxt.gs, nxt.es, j, n_exec, n_gen);
            if (j == n_exec - 1) last = cur.ee - cur.es;
            cur = nxt;
        }
    }
}

// Python `int / int` is the correctly rounded quotient; for |operands| < 2^53
// both convert exactly and IEEE division gives the same double.
__device__ __forceinline__ double wait_ratio(int64_t total, int64_t t_start, int64_t now,
                                             uint32_t* flag_bits) {
    if (now <= t_start) return 0.0;
    int64_t life = now - t_start;
    const int64_t lim = int64_t(1) << 53;
    if (total >= lim || total <= -lim || life >= lim) *flag_bits |= KR_FLAG_RATIO;
    // 0 / life = 0.0 exactly; a zero numerator is also outside the division's
    // fast-path range, and one such lane sent the whole warp through the slow
    // path (~90 instructions per request in the urgency pass)
    if (total == 0) return 0.0;
    double r = ddiv(static_cast<double>(total), static_cast<double>(life));
    r = r > 0.0 ? r : 0.0;
    return r < 1.0 ? r : 1.0;
}

__device__ __forceinline__ int32_t assign_bucket(double wr, int64_t skipped, int32_t B,
                                                 int32_t A) {
    int64_t b = static_cast<int64_t>(floor(dmul(wr, static_cast<double>(B))));
    if (b > B - 1) b = B - 1;
    if (skipped >= A) {
        b = b + skipped / A;
        if (b > B - 1) b = B - 1;
    }
    return static_cast<int32_t>(b);
}

// ---------------------------------------------------------------------------
// Packed composite key (ascending order == reference order)
//   kairos: hi = (B-1-b) << 56 | (2^56-1 - aged)      (scheduler.py:113-115,
//           lo = (issued - base) << 24 | lexrank        buckets high -> low)
//   fifo:   hi = issued ^ 2^63,  lo = lexrank          (scheduler.py:143-144)
//   las:    hi = accum_gen ^ 2^63, lo = (issued - base) << 24 | lexrank
// ---------------------------------------------------------------------------
constexpr uint64_t kAgedMask = (uint64_t(1) << 56) - 1;
constexpr int64_t kIssuedSpan = int64_t(1) << 40;
constexpr int64_t kRankSpan = int64_t(1) << 24;

__device__ __forceinline__ uint64_t issued_rank_word(int64_t issued, int64_t base, int32_t rank,
                                                     uint32_t* flag_bits) {
    int64_t d = issued - base;
    if (d < 0 || d >= kIssuedSpan || rank < 0 || rank >= kRankSpan) *flag_bits |= KR_FLAG_KEY_RANGE;
    return (static_cast<uint64_t>(d) << 24) | (static_cast<uint64_t>(rank) & 0xFFFFFFull);
}

__device__ __forceinline__ bool key_le(const kr_key& a, const kr_key& b) {
    return a.hi < b.hi || (a.hi == b.hi && a.lo <= b.lo);
}
__device__ __forceinline__ bool key_lt(const kr_key& a, const kr_key& b) {
    return a.hi < b.hi || (a.hi == b.hi && a.lo < b.lo);
}

// 128-bit logical right shift of (hi:lo) by s in [0, 127].
__device__ __forceinline__ uint64_t shr128_lo(uint64_t hi, uint64_t lo, int s) {
    if (s == 0) return lo;
    if (s < 64) return (lo >> s) | (hi << (64 - s));
    return hi >> (s - 64);
}

}  // namespace kr
