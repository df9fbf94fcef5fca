// kr_plan.cuh -- host-side launch planning shared by the streaming kernels
// (kr_horizon.cu, kr_sweep.cu): tile shape / ring depth / residency search
// and the cached launcher.
#pragma once

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <unordered_map>

#include "kr_host.cuh"
#include "kr_stream.cuh"

namespace kr {

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
                            int force_tr = 0, int max_stages = kMaxStages) {
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
    static const int tr_override = std::getenv("KR_PLAN_FORCE_TR")
                                       ? std::atoi(std::getenv("KR_PLAN_FORCE_TR")) : 0;
    if (tr_override > 0 && force_tr == 0) force_tr = tr_override;  // debug knob (sweeps)
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
            const uint64_t budget = smem_sm / per_sm - 1024 - 128 - kStreamStaticSmem;  // 1 KB reserved per CTA
            if (aux + 2 * sb <= budget) break;
        }
        if (per_sm < 1) continue;
        const uint64_t budget = smem_sm / per_sm - 1024 - 128 - kStreamStaticSmem;
        int stages = static_cast<int>((budget - aux) / sb);
        stages = stages > max_stages ? max_stages : stages;
        static const int max_stages_env = std::getenv("KR_PLAN_MAX_STAGES")
                                              ? std::atoi(std::getenv("KR_PLAN_MAX_STAGES")) : 0;
        if (max_stages_env >= 2 && stages > max_stages_env) stages = max_stages_env;  // debug knob
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

// Tile counters of the dynamic schedule (kr_stream.cuh stream_run): one
// {claimed, done} pair per launch captured into a CUDA graph, never reused (a
// replayed graph keeps its pair, and no two graphs -- nor a graph and another
// launch -- can ever share one, however they overlap); each launch's last CTA
// zeroes its pair, so every replay starts from zero.  Eager launches keep the
// static schedule; a process that captures more than kStreamCtrSlots launches
// per library unit falls back to it too.
constexpr int kStreamCtrSlots = 4096;
static __device__ unsigned g_stream_ctr[2 * kStreamCtrSlots];
static unsigned* stream_counters(cudaStream_t st) {
    // the pool's address is resolved by a launch outside capture (an eager
    // warm-up); a capture before any such launch keeps the static schedule
    static std::atomic<unsigned*> base{nullptr};
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess) return nullptr;
    if (cs == cudaStreamCaptureStatusNone) {
        if (!base.load()) {
            void* p = nullptr;
            if (cudaGetSymbolAddress(&p, g_stream_ctr) == cudaSuccess)
                base.store(static_cast<unsigned*>(p));
        }
        return nullptr;
    }
    if (cs != cudaStreamCaptureStatusActive || !base.load()) return nullptr;
    static std::atomic<unsigned> next{0};
    const unsigned k = next.fetch_add(1);
    return k < static_cast<unsigned>(kStreamCtrSlots) ? base.load() + 2 * k : nullptr;
}
static bool dynamic_tiles() {
    static const bool off = std::getenv("KR_STATIC_TILES") != nullptr;  // A/B knob
    return !off;
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
        if (p.max_per_sm > 0 && per_sm > p.max_per_sm) per_sm = p.max_per_sm;
        if (per_sm < 1) per_sm = 1;
        // sharing the GPU (max_sms > 0): one CTA slot per SM stays free so the
        // side stream's kernels can co-reside where registers are the limit.
        // max_sms < 0: cap at -max_sms SMs with every slot used (kernels whose
        // own footprint already leaves room, e.g. the segmented decide kernel)
        static const bool keep_slot = std::getenv("KR_SHARED_FULL_SM") == nullptr;  // A/B knob
        if (max_sms > 0 && keep_slot && per_sm > 1) per_sm -= 1;
        if (max_sms < 0) max_sms = -max_sms;
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
        StreamPlan pd = p;
        // the dynamic tail needs several tiles per CTA to balance (configs[1],
        // 1k robots, one tile per CTA: +2 us from the claims alone)
        if (p.mode == kModeBulk && !p.static_tiles && dynamic_tiles() && ntiles >= 8 * grid &&
            ntiles < (int64_t(1) << 31))
            pd.ctr = stream_counters(st);
        kern<<<static_cast<unsigned>(grid), p.threads + 32, smem, st>>>(pd, w, extra...);
        return check_launch(name);
    };
    return p.mode == kModeDirect ? go(kdirect) : go(kstaged);
}

}  // namespace kr
