// kr_stream.cuh -- persistent, TMA-fed streaming pipeline over fleet-major
// tensors.
//
// The horizon kernels read each robot's block exactly once: a contiguous byte
// range per input tensor (segment: the action rows, plus small per-robot
// metadata arrays such as the overlap offset, which therefore arrive in shared
// memory together with the rows they describe).  A tile is TR consecutive
// robots, i.e. one contiguous range per segment, so one elected thread moves a
// whole tile into shared memory with one `cp.async.bulk` (1-D TMA) per
// segment, completion tracked by a per-stage mbarrier.  STAGES tiles are in
// flight per CTA while the CTA's threads score the tile that already landed.
// The block size is matched to the tile: each thread owns the same few
// (robot slot, column/action) positions of every tile, so no index arithmetic
// runs per tile.  CTAs loop over tiles round-robin (grid = SMs x resident CTAs).
//
// Fallbacks: a base pointer that is not 16-byte aligned (or a tile that is not
// a multiple of 16 bytes) stages with plain loads; a robot too large for two
// stages of shared memory is scored straight from global memory.
#pragma once

#include "kr_common.cuh"

namespace kr {

constexpr int kMaxSeg = 5;
constexpr int kMaxRounds = 4;      // item positions per thread per tile
constexpr int kStreamThreads = 1024;
constexpr int kMaxStages = 8;      // ring depth (mbarrier slots)
constexpr int kStreamStaticSmem = 64;  // stream_run's static shared memory (dynamic tile ids)
#ifndef KR_DYN_TAIL_DIV
#define KR_DYN_TAIL_DIV 8  // the last ~1/8 of the tiles are claimed dynamically
#endif

// Segments have fixed slots (unused slots: rbytes 0) so that every segment
// pointer is a compile-time-indexed register, never a local-memory array.
struct StreamPlan {
    const unsigned char* base[kMaxSeg];  // global base of each segment
    uint32_t rbytes[kMaxSeg];            // bytes per robot in each segment (0: unused slot)
    uint32_t soff[kMaxSeg];              // offset of each segment in a stage buffer
    uint32_t stage_bytes;                // bytes per stage buffer (multiple of 128)
    uint32_t aux_bytes;                  // per-CTA scratch (after the mbarriers)
    int nseg;
    int TR;                              // robots per tile
    int stages;
    int mode;                            // 0 = TMA bulk, 1 = plain staged, 2 = direct
    int threads;                         // consumer threads (the CTA adds one producer warp)
    int rounds;                          // ceil(TR * items_per_robot / threads) <= kMaxRounds
    int max_per_sm;                      // resident CTAs per SM cap (0: occupancy decides)
    int64_t R;
    unsigned* ctr;                       // TMA mode: {tiles claimed, CTAs done} (null: static)
    int static_tiles;                    // launcher hint: keep the static schedule
};

enum { kModeBulk = 0, kModePlain = 1, kModeDirect = 2 };

// Shared-memory layout: [full[8], empty[8] mbarriers (128 B)] [aux] [stages]
__host__ __device__ inline uint32_t stream_aux_offset() { return 128; }
__host__ __device__ inline uint32_t stream_buf_offset(const StreamPlan& p) {
    return (stream_aux_offset() + p.aux_bytes + 127u) & ~127u;
}
__host__ inline size_t stream_smem_bytes(const StreamPlan& p) {
    if (p.mode == kModeDirect) return stream_buf_offset(p);
    return stream_buf_offset(p) + static_cast<size_t>(p.stages) * p.stage_bytes;
}

__device__ __forceinline__ void stream_issue(const StreamPlan& p, unsigned char* buf,
                                             uint64_t* bar, int64_t local, uint64_t pol,
                                             int64_t tile = -1) {
    int64_t t = tile >= 0 ? tile : blockIdx.x + local * gridDim.x;
    int64_t r0 = t * p.TR;
    int64_t nr = p.R - r0 < p.TR ? p.R - r0 : p.TR;
    uint32_t total = 0;
#pragma unroll
    for (int g = 0; g < kMaxSeg; g++) total += static_cast<uint32_t>(nr * p.rbytes[g]) & ~15u;
    mbar_arrive_expect_tx(bar, total);
#pragma unroll
    for (int g = 0; g < kMaxSeg; g++) {
        uint32_t b16 = static_cast<uint32_t>(nr * p.rbytes[g]) & ~15u;
        if (b16) bulk_g2s(buf + p.soff[g], p.base[g] + r0 * p.rbytes[g], b16, bar, pol);
    }
}

// Copy [from, to) bytes of every segment of tile (r0, nr) with 4-byte words.
__device__ __forceinline__ void stream_copy_plain(const StreamPlan& p, unsigned char* buf,
                                                  int64_t r0, int64_t nr, bool tail_only) {
#pragma unroll
    for (int g = 0; g < kMaxSeg; g++) {
        if (p.rbytes[g] == 0) continue;
        uint32_t bytes = static_cast<uint32_t>(nr * p.rbytes[g]);
        uint32_t from = tail_only ? (bytes & ~15u) : 0u;
        const uint32_t* src = reinterpret_cast<const uint32_t*>(p.base[g] + r0 * p.rbytes[g]);
        uint32_t* dst = reinterpret_cast<uint32_t*>(buf + p.soff[g]);
        for (uint32_t w = from / 4 + threadIdx.x; w < bytes / 4; w += blockDim.x)
            dst[w] = __ldg(src + w);
    }
}

struct TileView {
    const unsigned char* seg[kMaxSeg];  // segment bases of robot r0 (shared or global)
};

// Work must provide:
//   __device__ void tile(const TileView& v, int64_t r0, int nr, int slot);
//   __device__ void finish(int64_t r0, int nr, int slot, int lane, int nlanes);
// `slot` is the ring slot of the tile (per-slot scratch such as first-trip
// indices is reused only when that slot is refilled).  kStaged selects shared-
// memory staging (TMA bulk or plain) at compile time so that the scoring loads
// compile to LDS; !kStaged reads global memory.
//
// TMA mode synchronises through mbarriers only: full[s] (TMA bytes landed) and
// empty[s] (every warp finished reading slot s).  Warp 0 waits on empty[s],
// finishes the tile (writes its outputs, resets the slot scratch) and refills
// the slot; the other warps run ahead to the next landed tile without a
// block-wide barrier.
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

template <bool kStaged, class Work>
__device__ __forceinline__ void stream_run(const StreamPlan& p, unsigned char* smem, Work& work) {
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + 8;
    unsigned char* bufs = smem + stream_buf_offset(p);
    const int64_t ntiles = (p.R + p.TR - 1) / p.TR;
    if (blockIdx.x >= ntiles) return;
    const int64_t nlocal = (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
    const bool bulk = kStaged && p.mode == kModeBulk;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int consumer_warps = p.threads >> 5;     // the last warp is the producer
    const bool producer = warp == consumer_warps;
    uint64_t pol = 0;
    if (bulk) {
        pol = policy_evict_first();
        if (threadIdx.x == 0) {
            for (int s = 0; s < p.stages; s++) {
                mbar_init(&full[s], 1);
                mbar_init(&empty[s], consumer_warps);
            }
            fence_mbar_init();
        }
        __syncthreads();
    }
    // fleets below 2^31 robots (always, in practice) keep the tile arithmetic in 32 bits
    const bool small = p.R < (int64_t(1) << 31);
    auto tile_of = [&](int64_t i, int64_t& r0, int& nr) {
        if (small) {
            const int r32 = (static_cast<int>(blockIdx.x) + static_cast<int>(i) * static_cast<int>(gridDim.x)) * p.TR;
            const int left = static_cast<int>(p.R) - r32;
            r0 = r32;
            nr = left < p.TR ? left : p.TR;
        } else {
            r0 = (blockIdx.x + i * gridDim.x) * p.TR;
            nr = static_cast<int>(p.R - r0 < p.TR ? p.R - r0 : p.TR);
        }
    };
    if (bulk && p.ctr) {
        // Dynamic tiles: the producer claims each tile from a grid-wide counter
        // when it (re)fills a slot and leaves its index in tid_s[slot] (or -1:
        // none left, the slot's full barrier completed without bytes), so CTAs
        // that start late -- their SM held by the side stream's kernels -- take
        // fewer tiles instead of finishing a fixed share last.  The last CTA
        // done claiming resets the counters for the next launch.
        __shared__ int tid_s[kMaxStages];
        static_assert(sizeof(tid_s) <= kStreamStaticSmem, "plan budget");
        const unsigned nt = static_cast<unsigned>(ntiles);
        // a static prefix (round-robin, no atomics) of whole rounds over the
        // grid, then the tail claimed from the counter
        const unsigned G = gridDim.x;
        const unsigned nstat = (nt - nt / KR_DYN_TAIL_DIV) / G;  // static tiles per CTA
        const unsigned tail0 = nstat * G;
        unsigned next_stat = 0;
        auto fill = [&](int slot) {  // producer lane 0
            const unsigned t = next_stat < nstat ? blockIdx.x + (next_stat++) * G
                                                 : tail0 + atomicAdd(p.ctr, 1u);
            if (t < nt) {
                tid_s[slot] = static_cast<int>(t);
                stream_issue(p, bufs + static_cast<size_t>(slot) * p.stage_bytes, &full[slot], 0, pol, t);
            } else {
                tid_s[slot] = -1;
                mbar_arrive(&full[slot]);
            }
        };
        auto tile_at = [&](int t, int64_t& r0, int& nr) {
            r0 = static_cast<int64_t>(t) * p.TR;
            nr = static_cast<int>(p.R - r0 < p.TR ? p.R - r0 : p.TR);
        };
        if (producer) {
            if (lane == 0)
                for (int s = 0; s < p.stages; s++) fill(s);
            __syncwarp();
            int s = 0;
            uint32_t phase = 0;
            for (;;) {
                const int t = *reinterpret_cast<volatile int*>(&tid_s[s]);
                if (t < 0) break;
                int64_t r0;
                int nr;
                tile_at(t, r0, nr);
                mbar_wait(&empty[s], phase);
                work.finish(r0, nr, s, lane, 32);
                __syncwarp();
                if (lane == 0) fill(s);
                __syncwarp();
                if (++s == p.stages) {
                    s = 0;
                    phase ^= 1u;
                }
            }
            if (lane == 0 && atomicAdd(p.ctr + 1, 1u) == gridDim.x - 1) {
                p.ctr[0] = 0;
                p.ctr[1] = 0;
            }
            return;
        }
        int s = 0;
        uint32_t phase = 0;
        for (;;) {
            mbar_wait(&full[s], phase);
            const int t = *reinterpret_cast<volatile int*>(&tid_s[s]);
            if (t < 0) break;
            int64_t r0;
            int nr;
            tile_at(t, r0, nr);
            unsigned char* buf = bufs + static_cast<size_t>(s) * p.stage_bytes;
            if (nr < p.TR) {  // last tile: sub-16-byte remainder by hand (generic-proxy writes)
                for (int g = 0; g < kMaxSeg; g++) {
                    if (p.rbytes[g] == 0) continue;
                    const uint32_t bytes = static_cast<uint32_t>(nr * p.rbytes[g]);
                    const uint32_t* src = reinterpret_cast<const uint32_t*>(p.base[g] + r0 * p.rbytes[g]);
                    uint32_t* dst = reinterpret_cast<uint32_t*>(buf + p.soff[g]);
                    for (uint32_t w = (bytes & ~15u) / 4 + threadIdx.x; w < bytes / 4; w += p.threads)
                        dst[w] = __ldg(src + w);
                }
                fence_proxy_async_smem();
                asm volatile("bar.sync 1, %0;" ::"r"(p.threads));  // consumer warps only
            }
            TileView v;
#pragma unroll
            for (int g = 0; g < kMaxSeg; g++) v.seg[g] = buf + p.soff[g];
            work.tile(v, r0, nr, s);
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
            if (++s == p.stages) {
                s = 0;
                phase ^= 1u;
            }
        }
        return;
    }
    if (bulk && producer) {
        // producer warp: fill the ring, then per tile wait until every consumer
        // warp has released the slot, finish the tile, refill the slot
        if (lane == 0) {
            int64_t pre = nlocal < p.stages ? nlocal : p.stages;
            for (int64_t i = 0; i < pre; i++)
                stream_issue(p, bufs + static_cast<size_t>(i) * p.stage_bytes, &full[i], i, pol);
        }
        int s = 0;
        uint32_t phase = 0;
        for (int64_t i = 0; i < nlocal; i++) {
            int64_t r0;
            int nr;
            tile_of(i, r0, nr);
            mbar_wait(&empty[s], phase);
            work.finish(r0, nr, s, lane, 32);
            __syncwarp();
            if (lane == 0 && i + p.stages < nlocal)
                stream_issue(p, bufs + static_cast<size_t>(s) * p.stage_bytes, &full[s],
                             i + p.stages, pol);
            if (++s == p.stages) {
                s = 0;
                phase ^= 1u;
            }
        }
        return;
    }
    int s = 0;           // ring slot of tile i
    uint32_t phase = 0;  // mbarrier parity of that slot's current fill
    for (int64_t i = 0; i < nlocal; i++) {
        int64_t r0;
        int nr;
        tile_of(i, r0, nr);
        unsigned char* buf = bufs + static_cast<size_t>(s) * p.stage_bytes;
        TileView v;
        if constexpr (!kStaged) {
#pragma unroll
            for (int g = 0; g < kMaxSeg; g++) v.seg[g] = p.base[g] + r0 * p.rbytes[g];
            work.tile(v, r0, nr, 0);
            __syncthreads();
            work.finish(r0, nr, 0, threadIdx.x, blockDim.x);
            __syncthreads();
        } else if (!bulk) {  // plain staging: one buffer, block barriers
            stream_copy_plain(p, buf, r0, nr, false);
            __syncthreads();
#pragma unroll
            for (int g = 0; g < kMaxSeg; g++) v.seg[g] = buf + p.soff[g];
            work.tile(v, r0, nr, 0);
            __syncthreads();
            work.finish(r0, nr, 0, threadIdx.x, blockDim.x);
            __syncthreads();
        } else {
            mbar_wait(&full[s], phase);
            if (nr < p.TR) {  // last tile: sub-16-byte remainder by hand (generic-proxy writes)
                for (int g = 0; g < kMaxSeg; g++) {
                    if (p.rbytes[g] == 0) continue;
                    const uint32_t bytes = static_cast<uint32_t>(nr * p.rbytes[g]);
                    const uint32_t* src = reinterpret_cast<const uint32_t*>(p.base[g] + r0 * p.rbytes[g]);
                    uint32_t* dst = reinterpret_cast<uint32_t*>(buf + p.soff[g]);
                    for (uint32_t w = (bytes & ~15u) / 4 + threadIdx.x; w < bytes / 4; w += p.threads)
                        dst[w] = __ldg(src + w);
                }
                fence_proxy_async_smem();
                asm volatile("bar.sync 1, %0;" ::"r"(p.threads));  // consumer warps only
            }
#pragma unroll
            for (int g = 0; g < kMaxSeg; g++) v.seg[g] = buf + p.soff[g];
            work.tile(v, r0, nr, s);
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        }
        if (++s == p.stages) {
            s = 0;
            phase ^= 1u;
        }
    }
}

// First flagged index per robot for one round of items.  Items are ordered
// (robot, sample, index), so the lanes of a warp that score the same row
// (`run` = robot * S + sample) form one contiguous run with increasing index;
// the lowest flagged lane of a run carries the run's smallest index and is the
// only lane that touches shared memory.  Must be called by all 32 lanes.
__device__ __forceinline__ void first_flag(int* f, int rr, int run, bool flag, int idx) {
    const unsigned lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1;
    const int prev_run = __shfl_up_sync(0xffffffffu, run, 1);
    const unsigned bnd = __ballot_sync(0xffffffffu, lane == 0 || prev_run != run);
    const unsigned fb = __ballot_sync(0xffffffffu, flag);
    if (flag) {
        const unsigned run_lo = 31 - __clz(bnd & (lt | (1u << lane)));  // my run's first lane
        const unsigned below = lt & ~((1u << run_lo) - 1);              // run lanes below me
        if ((fb & below) == 0) atomicMin(&f[rr], idx);
    }
}

}  // namespace kr
