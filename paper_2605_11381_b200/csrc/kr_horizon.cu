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
#include <mutex>
#include <unordered_map>

#include "kr_common.cuh"
#include "kr_host.cuh"
#include "kr_stream.cuh"

namespace kr {

// ---------------------------------------------------------------------------
// Confidence threshold (horizon.py:108-132)
// ---------------------------------------------------------------------------
template <typename T, int KC>
struct ConfWork {
    int K, N, TR, hmin, rounds;
    double opt;   // 1.0 + threshold, rounded on the host as Python does
    float c1;     // (float)(opt / (K - 1)): the fp32 filter's mean-and-scale factor
    int32_t* H;
    uint32_t* flags;
    int* first;                  // [kMaxStages][TR] first tripping column per robot
    int rr_q[kMaxRounds];        // this thread's robot slot per round (-1: none)
    int n_q[kMaxRounds];         // ... and column

    __device__ void setup(int threads) {
        for (int q = 0; q < kMaxRounds; q++) {
            const int j = threadIdx.x + q * threads;
            const bool ok = q < rounds && j < TR * N && static_cast<int>(threadIdx.x) < threads;
            rr_q[q] = ok ? j / N : -1;
            n_q[q] = ok ? j - (j / N) * N : 0;
        }
    }

    // Exact fp32 pre-decision of `f > opt * mean` (fp32 storage): all terms are
    // non-negative, so the fp32 threshold sum * c1 is within (K + 8) * 2^-24 of
    // the exact one relative; undecided (or sub-1e-30 / overflowing) columns
    // use the bit-exact fp64 path.
    __device__ __forceinline__ int filter(float sf, float fin) const {
        if (fin == 0.f) return 0;  // 0 > thr is false for any thr >= 0
        const float thr = __fmul_rn(sf, c1);
        if (thr == 0.f) return sf == 0.f ? 1 : -1;  // exact zero mean: any f > 0 trips
        if (!(thr >= 1e-30f && thr <= 1e30f)) return -1;
        const float margin = static_cast<float>(K + 8) * 5.9604645e-8f;
        if (fin > thr * (1.f + margin)) return 1;
        if (fin < thr * (1.f - margin)) return 0;
        return -1;
    }

    __device__ __forceinline__ bool exact(const T* col) const {
        // u[:-1].mean(axis=0): sequential column add for N >= 2, numpy
        // pairwise summation when the reduction collapses (N == 1).
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
        return to_f64(col[static_cast<size_t>(K1) * N]) > dmul(opt, m);  // strict '>'
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
            bool trip = false;
            if (valid) {
                const int n = n_q[q];
                const T* col = u + static_cast<size_t>(rr) * Kr * N + n;
                // one pass over the column: validation (horizon.py:47-50) + fp32 sums
                float sf = 0.f, fin = 0.f;
                if constexpr (KC > 0) {
                    T x[KC];
#pragma unroll
                    for (int k = 0; k < KC; k++) x[k] = col[static_cast<size_t>(k) * N];
#pragma unroll
                    for (int k = 0; k < KC; k++) {
                        if (!isfinite(x[k])) fl |= KR_FLAG_NONFINITE;
                        if (x[k] < T(0)) fl |= KR_FLAG_NEGATIVE;
                    }
                    sf = static_cast<float>(x[0]);
#pragma unroll
                    for (int k = 1; k < KC - 1; k++) sf = __fadd_rn(sf, static_cast<float>(x[k]));
                    fin = static_cast<float>(x[KC - 1]);
                } else {
                    for (int k = 0; k < Kr; k++) {
                        const T x = col[static_cast<size_t>(k) * N];
                        if (!isfinite(x)) fl |= KR_FLAG_NONFINITE;
                        if (x < T(0)) fl |= KR_FLAG_NEGATIVE;
                        if (k == 0) sf = static_cast<float>(x);
                        else if (k < Kr - 1) sf = __fadd_rn(sf, static_cast<float>(x));
                        else fin = static_cast<float>(x);
                    }
                }
                int t = sizeof(T) == 4 ? filter(sf, fin) : -1;
                if (t < 0) t = exact(col);
                trip = t;
            }
            first_flag(f, valid ? rr : -1, valid ? rr : -1, trip, n_q[q]);
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

template <typename T, int KC, bool kStaged>
__global__ void __launch_bounds__(kStreamThreads) k_horizon_confidence(StreamPlan p, ConfWork<T, KC> w) {
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
template <typename T, int DC>
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
        const int per = S * Lc;
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

    __device__ __forceinline__ void tile(const TileView& v, int64_t r0, int nr, int slot) {
        const T* prev = reinterpret_cast<const T*>(v.seg[0]);
        const T* cand = reinterpret_cast<const T*>(v.seg[1]);
        int* f = first + slot * TR;
        int* lm = lim + slot * TR;
        const int D_ = DC > 0 ? DC : D;
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

template <typename T, int DC, bool kStaged>
__global__ void __launch_bounds__(div_max_threads<DC>()) k_horizon_divergence(StreamPlan p,
                                                                             DivWork<T, DC> w) {
    extern __shared__ __align__(128) unsigned char smem[];
    w.first = reinterpret_cast<int*>(smem + stream_aux_offset());
    w.lim = w.first + kMaxStages * w.TR;
    for (int i = threadIdx.x; i < kMaxStages * w.TR; i += blockDim.x) w.first[i] = INT_MAX;
    w.setup(p.threads);
    __syncthreads();
    stream_run<kStaged>(p, smem, w);
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
                            int regs_per_thread) {
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
    const int regs = ((regs_per_thread > 0 ? regs_per_thread : 64) + 7) / 8 * 8;
    const uint64_t smem_sm = static_cast<uint64_t>(di.max_smem_optin) + 1024;  // per-SM pool
    const double kInflightTarget = 160.0 * 1024;
    double best = 1e30;
    for (int64_t t = 1; t <= 1024; t++) {
        const int64_t items = t * items_per_robot;
        if (items > static_cast<int64_t>(max_threads) * kMaxRounds) break;
        const int rounds = static_cast<int>((items + max_threads - 1) / max_threads);
        const int threads = static_cast<int>(((items + rounds - 1) / rounds + 31) / 32 * 32);
        const uint64_t sb = stage_bytes(t);
        const uint64_t aux = (256 + t * aux_per_robot + 127) & ~uint64_t(127);
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
        p.aux_bytes = 256 + aux_per_robot;
        p.stage_bytes = 0;
        return p;
    }
    p.aux_bytes = static_cast<uint32_t>(256 + p.TR * aux_per_robot);
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

template <class Work, class KStaged, class KDirect>
static int launch_stream(KStaged kstaged, KDirect kdirect, const StreamPlan& p, const Work& w,
                         cudaStream_t st, const char* name, int max_sms = 0) {
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
        kern<<<static_cast<unsigned>(grid), p.threads + 32, smem, st>>>(p, w);
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
        StreamPlan p = make_plan(1, bases, &rb, R, N, kMaxStages * sizeof(int), kStreamThreads - 32,
                                 kernel_regs(kstaged));
        W w{K, N, p.TR, min_horizon, p.rounds, one_plus_t, c1, H, flags, nullptr, {}, {}};
        return launch_stream(kstaged, kdirect, p, w, st, "kr_horizon_confidence");
    };
    if (dtype == KR_F64) {
        if (K == 6)
            return go(ConfWork<double, 6>{}, k_horizon_confidence<double, 6, true>,
                      k_horizon_confidence<double, 6, false>);
        return go(ConfWork<double, 0>{}, k_horizon_confidence<double, 0, true>,
                  k_horizon_confidence<double, 0, false>);
    }
    if (K == 6)
        return go(ConfWork<float, 6>{}, k_horizon_confidence<float, 6, true>,
                  k_horizon_confidence<float, 6, false>);
    return go(ConfWork<float, 0>{}, k_horizon_confidence<float, 0, true>,
              k_horizon_confidence<float, 0, false>);
}

template <typename T>
static int launch_div(const StreamPlan& p, const DivWork<T, 0>& w0, cudaStream_t st, int max_sms) {
    auto with = [&](auto proto) {
        decltype(proto) w{w0.S, w0.Lp, w0.Lc, w0.D, w0.TR, w0.rounds, w0.has_off, w0.has_lp,
                          w0.has_lc, w0.thr, w0.H, w0.cos, w0.thr_f, w0.margin, nullptr, nullptr,
                          {}, {}, {}};
        return w;
    };
    switch (w0.D) {
        case 7:
            return launch_stream(k_horizon_divergence<T, 7, true>, k_horizon_divergence<T, 7, false>,
                                 p, with(DivWork<T, 7>{}), st, "kr_horizon_divergence", max_sms);
        case 32:
            return launch_stream(k_horizon_divergence<T, 32, true>,
                                 k_horizon_divergence<T, 32, false>, p, with(DivWork<T, 32>{}), st,
                                 "kr_horizon_divergence", max_sms);
        default:
            return launch_stream(k_horizon_divergence<T, 0, true>, k_horizon_divergence<T, 0, false>,
                                 p, w0, st, "kr_horizon_divergence", max_sms);
    }
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
    if (static_cast<int64_t>(S) * Lc > static_cast<int64_t>(kStreamThreads) * kMaxRounds)
        return KR_EINVAL;
    // segments: action rows, then the per-robot metadata that travels with them
    const void* bases[5] = {prev, cand, offset, len_prev, len_cand};
    uint64_t rbs[5] = {rb[0], rb[1], offset ? 4u : 0u, len_prev ? 4u : 0u, len_cand ? 4u : 0u};
    const int nseg = 5;
    const int maxt = D == 7 ? kStreamThreads : 256;  // only D = 7 has a small-D kernel
    if (static_cast<int64_t>(S) * Lc > static_cast<int64_t>(maxt - 32) * kMaxRounds) return KR_EINVAL;
    int regs;
    if (dtype == KR_F64)
        regs = D == 7 ? kernel_regs(k_horizon_divergence<double, 7, true>)
                      : (D == 32 ? kernel_regs(k_horizon_divergence<double, 32, true>)
                                 : kernel_regs(k_horizon_divergence<double, 0, true>));
    else
        regs = D == 7 ? kernel_regs(k_horizon_divergence<float, 7, true>)
                      : (D == 32 ? kernel_regs(k_horizon_divergence<float, 32, true>)
                                 : kernel_regs(k_horizon_divergence<float, 0, true>));
    StreamPlan p = make_plan(nseg, bases, rbs, R, S * Lc, 2 * kMaxStages * sizeof(int), maxt - 32,
                             regs);
    cudaStream_t st = as_stream(stream);
    const float thr_f = static_cast<float>(thr);
    const float margin = cos_filter_margin(D);
    if (dtype == KR_F64) {
        DivWork<double, 0> w{S, Lp, Lc, D, p.TR, p.rounds, offset != nullptr, len_prev != nullptr,
                             len_cand != nullptr, thr, H, cos, thr_f, margin, nullptr, nullptr,
                             {}, {}, {}};
        return launch_div(p, w, st, max_sms);
    }
    DivWork<float, 0> w{S, Lp, Lc, D, p.TR, p.rounds, offset != nullptr, len_prev != nullptr,
                        len_cand != nullptr, thr, H, cos, thr_f, margin, nullptr, nullptr,
                        {}, {}, {}};
    return launch_div(p, w, st, max_sms);
}
