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

#include "kr_common.cuh"
#include "kr_host.cuh"
#include "kr_stream.cuh"

namespace kr {

// Warp-aggregated "first index" update: lanes scoring the same robot combine
// their candidate indices with one shuffle-reduction; one lane per robot
// touches shared memory.
__device__ __forceinline__ void first_min(int* f, int rr, int idx) {
    const unsigned active = __activemask();
    const unsigned peers = __match_any_sync(active, rr);
    const int m = __reduce_min_sync(peers, idx);
    if (m != INT_MAX && (threadIdx.x & 31) == __ffs(peers) - 1) atomicMin(&f[rr], m);
}

// ---------------------------------------------------------------------------
// Confidence threshold (horizon.py:108-132)
// ---------------------------------------------------------------------------
template <typename T>
struct ConfWork {
    int K, N, TR, hmin;
    double opt;  // 1.0 + threshold, rounded on the host as Python does
    int32_t* H;
    uint32_t* flags;
    FastDiv divN;
    int* first;  // [2][TR] first tripping column per robot, INT_MAX = none

    // Exact fp32 pre-decision of `f > opt * mean` for fp32 storage: all terms
    // are non-negative, so the fp32 threshold is within (K + 8) * 2^-24 of the
    // exact one relative; undecided (or sub-1e-30 / overflowing) columns use
    // the bit-exact fp64 path.
    __device__ __forceinline__ int filter(const T* col) const {
        if constexpr (sizeof(T) != 4) {
            return -1;
        } else {
            float sf = col[0];
            for (int k = 1; k < K - 1; k++) sf = __fadd_rn(sf, col[static_cast<size_t>(k) * N]);
            const float fin = col[static_cast<size_t>(K - 1) * N];
            if (fin == 0.f) return 0;  // 0 > thr is false for any thr >= 0
            const float thr = __fmul_rn(__fdiv_rn(sf, static_cast<float>(K - 1)),
                                        static_cast<float>(opt));
            if (thr == 0.f) return sf == 0.f ? 1 : -1;  // exact zero mean: any f > 0 trips
            if (!(thr >= 1e-30f && thr <= 1e30f)) return -1;
            const float margin = static_cast<float>(K + 8) * 5.9604645e-8f;
            if (fin > thr * (1.f + margin)) return 1;
            if (fin < thr * (1.f - margin)) return 0;
            return -1;
        }
    }

    __device__ void tile(const unsigned char* seg0, const unsigned char*, int64_t, int nr,
                         int64_t local) {
        const T* u = reinterpret_cast<const T*>(seg0);
        int* f = first + (local & 1) * TR;
        uint32_t fl = 0;
        const int K1 = K - 1;
        const double dK1 = static_cast<double>(K1);
        const int items = nr * N;
        for (int j = threadIdx.x; j < items; j += blockDim.x) {
            const int rr = static_cast<int>(fdiv(static_cast<uint32_t>(j), divN));
            const int n = j - rr * N;
            const T* col = u + static_cast<size_t>(rr) * K * N + n;
            // Validation (horizon.py:47-50) covers every element of the round.
            for (int k = 0; k < K; k++) {
                T v = col[static_cast<size_t>(k) * N];
                if (!isfinite(v)) fl |= KR_FLAG_NONFINITE;
                if (v < T(0)) fl |= KR_FLAG_NEGATIVE;
            }
            int trip = filter(col);
            if (trip < 0) {
                // u[:-1].mean(axis=0): sequential column add for N >= 2, numpy
                // pairwise summation when the reduction collapses (N == 1).
                double s;
                if (N >= 2) {
                    s = to_f64(col[0]);
                    for (int k = 1; k < K1; k++) s = dadd(s, to_f64(col[static_cast<size_t>(k) * N]));
                } else {
                    auto a = [col](int64_t k) { return to_f64(col[k]); };
                    s = np_pairwise_sum(a, 0, K1);
                }
                double m = ddiv(s, dK1);
                double fin = to_f64(col[static_cast<size_t>(K1) * N]);
                trip = fin > dmul(opt, m);  // strict '>' (horizon.py:127)
            }
            first_min(f, rr, trip ? n : INT_MAX);
        }
        if (fl && flags) atomicOr(flags, fl);
    }

    __device__ void finish(int64_t r0, int nr, int64_t local) {
        int* f = first + (local & 1) * TR;
        for (int rr = threadIdx.x; rr < nr; rr += blockDim.x) {
            int h = f[rr] < N ? f[rr] : N;  // argmax of trips, or N
            h = h > hmin ? h : hmin;
            H[r0 + rr] = h < N ? h : N;
            f[rr] = INT_MAX;
        }
    }
};

template <typename T>
__global__ void __launch_bounds__(kMaxThreads) k_horizon_confidence(StreamPlan p, ConfWork<T> w) {
    extern __shared__ __align__(128) unsigned char smem[];
    w.first = reinterpret_cast<int*>(smem + stream_aux_offset());
    for (int i = threadIdx.x; i < 2 * w.TR; i += blockDim.x) w.first[i] = INT_MAX;
    __syncthreads();
    stream_run(p, smem, w);
}

// ---------------------------------------------------------------------------
// Divergence horizon (workload.py:461-496), S-sample ensembles, ragged rows
// ---------------------------------------------------------------------------
template <typename T, int DC>
struct DivWork {
    int S, Lp, Lc, D, TR;
    const int32_t *off, *lenp, *lenc;
    double thr;
    int32_t* H;
    double* cos;
    FastDiv divRobot, divLc;  // S * Lc, Lc
    float thr_f, margin;
    int* first;  // [2][TR]
    int2* meta;  // [2][TR] (offset, limit) of each robot of the tile

    __device__ __forceinline__ int2 load_meta(int64_t r) const {
        int o = off ? __ldg(off + r) : 0;
        int lp = lenp ? __ldg(lenp + r) : Lp;
        int lc = lenc ? __ldg(lenc + r) : Lc;
        o = o < 0 ? 0 : o;
        lp = lp > Lp ? Lp : lp;
        lc = lc > Lc ? Lc : (lc < 0 ? 0 : lc);
        int lr = lp - o;
        lr = lr < 0 ? 0 : lr;
        return make_int2(o, lr < lc ? lr : lc);
    }

    __device__ void tile(const unsigned char* seg0, const unsigned char* seg1, int64_t r0, int nr,
                         int64_t local) {
        const T* prev = reinterpret_cast<const T*>(seg0);
        const T* cand = reinterpret_cast<const T*>(seg1);
        int* f = first + (local & 1) * TR;
        int2* mt = meta + (local & 1) * TR;
        for (int rr = threadIdx.x; rr < nr; rr += blockDim.x) mt[rr] = load_meta(r0 + rr);
        __syncthreads();
        const int D_ = DC > 0 ? DC : D;
        const int items = nr * S * Lc;
        for (int j = threadIdx.x; j < items; j += blockDim.x) {
            const int rr = static_cast<int>(fdiv(static_cast<uint32_t>(j), divRobot));
            const int rem = j - rr * S * Lc;
            const int s = static_cast<int>(fdiv(static_cast<uint32_t>(rem), divLc));
            const int i = rem - s * Lc;
            const int2 m = mt[rr];
            int fail = INT_MAX;
            if (i < m.y) {
                const T* a = cand + (static_cast<size_t>(rr * S + s) * Lc + i) * D_;
                const T* b = prev + (static_cast<size_t>(rr) * Lp + m.x + i) * D_;
                int pass = -1;
                if (!cos) {
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
                    if (cos) cos[(static_cast<size_t>(r0 + rr) * S + s) * Lc + i] = c;
                }
                if (!pass) fail = i;  // first action below threshold ends the prefix
            } else if (cos) {
                cos[(static_cast<size_t>(r0 + rr) * S + s) * Lc + i] =
                    __longlong_as_double(0x7ff8000000000000LL);  // NaN past the limit
            }
            first_min(f, rr, fail);
        }
    }

    __device__ void finish(int64_t r0, int nr, int64_t local) {
        int* f = first + (local & 1) * TR;
        const int2* mt = meta + (local & 1) * TR;
        for (int rr = threadIdx.x; rr < nr; rr += blockDim.x) {
            const int limit = mt[rr].y;
            H[r0 + rr] = f[rr] < limit ? f[rr] : limit;
            f[rr] = INT_MAX;
        }
    }
};

template <typename T, int DC>
__global__ void __launch_bounds__(kMaxThreads) k_horizon_divergence(StreamPlan p, DivWork<T, DC> w) {
    extern __shared__ __align__(128) unsigned char smem[];
    w.first = reinterpret_cast<int*>(smem + stream_aux_offset());
    w.meta = reinterpret_cast<int2*>(smem + stream_aux_offset() + 2 * w.TR * sizeof(int));
    for (int i = threadIdx.x; i < 2 * w.TR; i += blockDim.x) w.first[i] = INT_MAX;
    __syncthreads();
    stream_run(p, smem, w);
}

__global__ void k_horizon_static(int64_t R, int32_t h, int32_t* H) {
    for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < R;
         r += int64_t(gridDim.x) * blockDim.x)
        H[r] = h;
}

// ---------------------------------------------------------------------------
// Launch planning
// ---------------------------------------------------------------------------
// Tile sizing.  A tile is TR robots; its work items (columns / actions) are
// spread over the CTA's threads, so TR is chosen to keep the last round of
// items nearly full, each stage 8-48 KB, TMA-alignable (TR * row bytes a
// multiple of 16) and the whole ring small enough for two CTAs per SM (16
// warps to hide the scoring latency; 3-4 stages keep >= 2 tiles in flight).
static StreamPlan make_plan(int nseg, const void* const* base, const uint64_t* rbytes, int64_t R,
                            int items_per_robot, uint32_t aux_per_robot) {
    const DeviceInfo& di = device_info();
    StreamPlan p{};
    p.nseg = nseg;
    p.R = R;
    bool base_ok = true;
    for (int g = 0; g < nseg; g++) {
        p.base[g] = static_cast<const unsigned char*>(base[g]);
        p.rbytes[g] = static_cast<uint32_t>(rbytes[g]);
        base_ok = base_ok && aligned16(base[g]);
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
    const uint64_t smem_max = static_cast<uint64_t>(di.max_smem_optin) - 1024;
    int best_tr = 0, best_stages = 0;
    double best_score = 1e30;
    for (int per_sm = 2; per_sm >= 1 && best_tr == 0; per_sm--) {
        const uint64_t budget = smem_max / per_sm - 1024;
        for (int64_t t = 1; t <= 1024 && t <= R + 1; t++) {
            const uint64_t sb = stage_bytes(t);
            const uint64_t aux = (256 + t * aux_per_robot + 127) & ~uint64_t(127);
            if (t > 1 && sb > 48 * 1024) break;
            if (2 * sb + aux > budget) break;
            int stages = static_cast<int>((budget - aux) / sb);
            stages = stages > 4 ? 4 : stages;
            const int64_t items = t * items_per_robot;
            const int64_t rounds = (items + kMaxThreads - 1) / kMaxThreads;
            double score = 1.0 - static_cast<double>(items) / (rounds * kMaxThreads);
            if (sb < 12 * 1024) score += 0.05;                 // tiny tiles: per-tile overhead
            if (!tma_ok(t)) score += 1.0;                       // plain staging is much slower
            if (score < best_score - 1e-9 || (score < best_score + 1e-9 && t > best_tr)) {
                best_score = score;
                best_tr = static_cast<int>(t);
                best_stages = stages;
            }
        }
    }
    if (best_tr == 0) {  // robot larger than two stages of shared memory: score from global
        p.TR = 1;
        p.stages = 1;
        p.mode = kModeDirect;
        p.aux_bytes = 256 + aux_per_robot;
        p.stage_bytes = 0;
        return p;
    }
    p.TR = best_tr;
    p.stages = best_stages;
    p.aux_bytes = static_cast<uint32_t>(256 + best_tr * aux_per_robot);
    uint32_t off = 0;
    for (int g = 0; g < nseg; g++) {
        p.soff[g] = off;
        off += static_cast<uint32_t>(((uint64_t)best_tr * rbytes[g] + 127) & ~uint64_t(127));
    }
    p.stage_bytes = off;
    p.mode = tma_ok(best_tr) ? kModeBulk : kModePlain;
    if (p.mode == kModePlain) p.stages = 1;
    return p;
}

template <class Kern, class Work>
static int launch_stream(Kern kern, const StreamPlan& p, const Work& w, cudaStream_t st,
                         const char* name) {
    size_t smem = stream_smem_bytes(p);
    KR_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem)));
    int per_sm = 0;
    KR_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kMaxThreads, smem));
    if (per_sm < 1) per_sm = 1;
    int64_t ntiles = (p.R + p.TR - 1) / p.TR;
    int64_t grid = static_cast<int64_t>(device_info().sm_count) * per_sm;
    if (grid > ntiles) grid = ntiles;
    if (grid < 1) grid = 1;
    kern<<<static_cast<unsigned>(grid), kMaxThreads, smem, st>>>(p, w);
    return check_launch(name);
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
    const void* bases[1] = {U};
    StreamPlan p = make_plan(1, bases, &rb, R, N, 2 * sizeof(int));
    cudaStream_t st = as_stream(stream);
    const FastDiv dN = make_fastdiv(static_cast<uint32_t>(N));
    if (dtype == KR_F64) {
        ConfWork<double> w{K, N, p.TR, min_horizon, one_plus_t, H, flags, dN, nullptr};
        return launch_stream(k_horizon_confidence<double>, p, w, st, "kr_horizon_confidence");
    }
    ConfWork<float> w{K, N, p.TR, min_horizon, one_plus_t, H, flags, dN, nullptr};
    return launch_stream(k_horizon_confidence<float>, p, w, st, "kr_horizon_confidence");
}

template <typename T>
static int launch_div(const StreamPlan& p, const DivWork<T, 0>& w0, cudaStream_t st) {
    switch (w0.D) {
        case 7: {
            DivWork<T, 7> w{w0.S, w0.Lp, w0.Lc, w0.D, w0.TR, w0.off, w0.lenp, w0.lenc,
                            w0.thr, w0.H, w0.cos, w0.divRobot, w0.divLc, w0.thr_f, w0.margin,
                            nullptr, nullptr};
            return launch_stream(k_horizon_divergence<T, 7>, p, w, st, "kr_horizon_divergence");
        }
        case 32: {
            DivWork<T, 32> w{w0.S, w0.Lp, w0.Lc, w0.D, w0.TR, w0.off, w0.lenp, w0.lenc,
                             w0.thr, w0.H, w0.cos, w0.divRobot, w0.divLc, w0.thr_f, w0.margin,
                             nullptr, nullptr};
            return launch_stream(k_horizon_divergence<T, 32>, p, w, st, "kr_horizon_divergence");
        }
        default:
            return launch_stream(k_horizon_divergence<T, 0>, p, w0, st, "kr_horizon_divergence");
    }
}

extern "C" int kr_horizon_divergence(const void* prev, const void* cand, int dtype, int64_t R,
                                     int32_t S, int32_t Lp, int32_t Lc, int32_t D,
                                     const int32_t* offset, const int32_t* len_prev,
                                     const int32_t* len_cand, double thr, int32_t* H, double* cos,
                                     void* stream) {
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
    const void* bases[2] = {prev, cand};
    StreamPlan p = make_plan(2, bases, rb, R, S * Lc, 2 * sizeof(int) + 2 * sizeof(int2));
    cudaStream_t st = as_stream(stream);
    const FastDiv dR = make_fastdiv(static_cast<uint32_t>(S * Lc));
    const FastDiv dL = make_fastdiv(static_cast<uint32_t>(Lc));
    const float thr_f = static_cast<float>(thr);
    const float margin = cos_filter_margin(D);
    if (dtype == KR_F64) {
        DivWork<double, 0> w{S, Lp, Lc, D, p.TR, offset, len_prev, len_cand, thr, H, cos,
                             dR, dL, thr_f, margin, nullptr, nullptr};
        return launch_div(p, w, st);
    }
    DivWork<float, 0> w{S, Lp, Lc, D, p.TR, offset, len_prev, len_cand, thr, H, cos,
                        dR, dL, thr_f, margin, nullptr, nullptr};
    return launch_div(p, w, st);
}
