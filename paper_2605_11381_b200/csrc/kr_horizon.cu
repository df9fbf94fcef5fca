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
                            int regs_per_thread, int min_rounds = 1) {
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
    for (int64_t t = 1; t <= 1024; t++) {
        const int64_t items = t * items_per_robot;
        if (items > static_cast<int64_t>(max_threads) * kMaxRounds) break;
        int rounds = static_cast<int>((items + max_threads - 1) / max_threads);
        if (rounds < min_rounds) {
            if (items < static_cast<int64_t>(min_rounds) * 32) continue;
            rounds = min_rounds;
        }
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
        static const bool trace = std::getenv("KR_TRACE_PLAN") != nullptr;
        if (trace)
            std::fprintf(stderr, "[kr plan] %s R=%lld TR=%d threads=%d+32 rounds=%d stages=%d "
                         "mode=%d stage_bytes=%u smem=%zu grid=%lld per_sm=%d\n", name,
                         static_cast<long long>(p.R), p.TR, p.threads, p.rounds, p.stages, p.mode,
                         p.stage_bytes, smem, static_cast<long long>(grid), per_sm);
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
