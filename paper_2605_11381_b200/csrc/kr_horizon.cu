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
#include <atomic>
#include <mutex>
#include <unordered_map>

#include "kr_common.cuh"
#include "kr_host.cuh"
#include "kr_stream.cuh"

#include "kr_conf.cuh"
#include "kr_div.cuh"
#include "kr_plan.cuh"
#include "kr_sweep.cuh"

namespace kr {

__global__ void k_horizon_static(int64_t R, int32_t h, int32_t* H) {
    for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < R;
         r += int64_t(gridDim.x) * blockDim.x)
        H[r] = h;
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
                                     uint32_t* flags, int32_t max_sms, void* stream) {
    if (R < 0 || K < 2 || N < 1 || min_horizon < 1 || (dtype != KR_F32 && dtype != KR_F64))
        return KR_EINVAL;
    if (R == 0) return KR_OK;
    if (!U || !H) return KR_EINVAL;
    const size_t es = dtype == KR_F64 ? 8 : 4;
    uint64_t rb = static_cast<uint64_t>(K) * N * es;
    if (N > (kStreamThreads - 32) * kMaxRounds) return KR_EINVAL;
    cudaStream_t st = as_stream(stream);
    // Default: the segmented decide kernel (kr_sweep.cuh SweepSeg) as a
    // one-configuration sweep writing H -- per robot a handful of lanes decide
    // register-resident column windows (a third of this kernel's instructions,
    // a third of its warps), which leaves SM slots for the round's side stream.
    // Thresholds whose bucket table cannot be built (1 + t beyond ~1e30) and
    // shapes the segmented layout does not take stay on k_horizon_confidence.
    static const bool classic = std::getenv("KR_CONF_CLASSIC") != nullptr;  // A/B knob
    // (fp32 storage only: with fp64 the round-1 kernel measured faster in the round)
    if (!classic && dtype == KR_F32 && one_plus_t >= 1.0 && one_plus_t < 1e30 &&
        sweep_seg_ok(K, N, es, (reinterpret_cast<uintptr_t>(U) & 15u) == 0)) {
        const int32_t kind = 1, param = min_horizon;
        SweepCfg cfg;
        if (sweep_make_cfg(dtype, K, N, 1, &kind, &one_plus_t, &param, cfg) == KR_OK &&
            cfg.lut_below == 0) {
            const int rc = dtype == KR_F64
                               ? sweep_run_f64(U, R, K, N, 1, cfg.Cc, cfg, nullptr, H, flags, st, max_sms)
                               : sweep_run_f32(U, R, K, N, 1, cfg.Cc, cfg, nullptr, H, flags, st, max_sms);
            if (rc != KR_EINVAL) return rc;
        }
    }
    const void* bases[1] = {U};
    const float c1 = static_cast<float>(one_plus_t / static_cast<double>(K - 1));
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
        return launch_stream(kstaged, kdirect, p, w, st, "kr_horizon_confidence", max_sms);
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

// Process-wide, like OpenBLAS' own core choice; read when a launch is set up
// (a captured CUDA graph keeps the order it was captured with).
static std::atomic<int> g_dot_order{kDotSkylakeX};

extern "C" int kr_set_dot_order(int32_t order) {
    if (order != KR_DOT_SKYLAKEX && order != KR_DOT_HASWELL) return KR_EINVAL;
    g_dot_order.store(order);
    return KR_OK;
}

extern "C" int32_t kr_get_dot_order(void) { return g_dot_order.load(); }

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
    const DivArgs a{prev, cand, dtype, R, S, Lp, Lc, D, offset, len_prev, len_cand, thr, H, cos,
                    max_sms, stream};
    return g_dot_order.load() == kDotHaswell ? div_run_hsw(a) : div_run_skx(a);
}
