// kr_stream.cuh -- persistent, TMA-fed streaming pipeline over fleet-major
// tensors.
//
// The horizon kernels read each robot's block exactly once: a contiguous byte
// range per input tensor (segment).  A tile is TR consecutive robots, i.e. one
// contiguous range per segment, so one elected thread moves a whole tile into
// shared memory with one `cp.async.bulk` (1-D TMA) per segment, completion
// tracked by a per-stage mbarrier.  STAGES tiles are in flight per CTA while the
// other threads score the tile that already landed; one CTA per SM slot loops
// over tiles round-robin (grid = SMs x resident CTAs).
//
// Fallbacks: a base pointer that is not 16-byte aligned (or a tile size that is
// not a multiple of 16 bytes) stages with plain loads; a robot too large for
// two stages of shared memory is scored straight from global memory.
#pragma once

#include "kr_common.cuh"

namespace kr {

constexpr int kMaxSeg = 2;

struct StreamPlan {
    const unsigned char* base[kMaxSeg];  // global base of each segment
    uint32_t rbytes[kMaxSeg];            // bytes per robot in each segment
    uint32_t soff[kMaxSeg];              // offset of each segment in a stage buffer
    uint32_t stage_bytes;                // bytes per stage buffer (multiple of 128)
    uint32_t aux_bytes;                  // per-CTA scratch (after the mbarriers)
    int nseg;
    int TR;                              // robots per tile
    int stages;
    int mode;                            // 0 = TMA bulk, 1 = plain staged, 2 = direct
    int64_t R;
};

enum { kModeBulk = 0, kModePlain = 1, kModeDirect = 2 };

// Shared-memory layout: [mbarriers (8 B x stages, padded to 128)] [aux] [stages]
__host__ __device__ inline uint32_t stream_aux_offset() { return 128; }
__host__ __device__ inline uint32_t stream_buf_offset(const StreamPlan& p) {
    return (stream_aux_offset() + p.aux_bytes + 127u) & ~127u;
}
__host__ inline size_t stream_smem_bytes(const StreamPlan& p) {
    if (p.mode == kModeDirect) return stream_buf_offset(p);
    return stream_buf_offset(p) + static_cast<size_t>(p.stages) * p.stage_bytes;
}

__device__ __forceinline__ void stream_issue(const StreamPlan& p, unsigned char* bufs,
                                             uint64_t* mbar, int64_t local, uint64_t pol) {
    int s = static_cast<int>(local % p.stages);
    int64_t t = blockIdx.x + local * gridDim.x;
    int64_t r0 = t * p.TR;
    int64_t nr = p.R - r0 < p.TR ? p.R - r0 : p.TR;
    unsigned char* buf = bufs + static_cast<size_t>(s) * p.stage_bytes;
    uint32_t total = 0;
#pragma unroll
    for (int g = 0; g < kMaxSeg; g++)
        if (g < p.nseg) total += static_cast<uint32_t>(nr * p.rbytes[g]) & ~15u;
    mbar_arrive_expect_tx(&mbar[s], total);
#pragma unroll
    for (int g = 0; g < kMaxSeg; g++) {
        if (g >= p.nseg) break;
        uint32_t b16 = static_cast<uint32_t>(nr * p.rbytes[g]) & ~15u;
        if (b16) bulk_g2s(buf + p.soff[g], p.base[g] + r0 * p.rbytes[g], b16, &mbar[s], pol);
    }
}

// Copy [from, to) bytes of every segment of tile (r0, nr) with 4-byte words.
__device__ __forceinline__ void stream_copy_plain(const StreamPlan& p, unsigned char* buf,
                                                  int64_t r0, int64_t nr, bool tail_only) {
#pragma unroll
    for (int g = 0; g < kMaxSeg; g++) {
        if (g >= p.nseg) break;
        uint32_t bytes = static_cast<uint32_t>(nr * p.rbytes[g]);
        uint32_t from = tail_only ? (bytes & ~15u) : 0u;
        const uint32_t* src = reinterpret_cast<const uint32_t*>(p.base[g] + r0 * p.rbytes[g]);
        uint32_t* dst = reinterpret_cast<uint32_t*>(buf + p.soff[g]);
        for (uint32_t w = from / 4 + threadIdx.x; w < bytes / 4; w += blockDim.x)
            dst[w] = __ldg(src + w);
    }
}

// Work must provide:
//   __device__ void tile(const unsigned char* seg0, const unsigned char* seg1,
//                        int64_t r0, int nr, int64_t local);
//   __device__ void finish(int64_t r0, int nr, int64_t local);
// `tile` sees the segment bases of robot r0 (shared or global memory).
template <class Work>
__device__ __forceinline__ void stream_run(const StreamPlan& p, unsigned char* smem, Work& work) {
    uint64_t* mbar = reinterpret_cast<uint64_t*>(smem);
    unsigned char* bufs = smem + stream_buf_offset(p);
    int64_t ntiles = (p.R + p.TR - 1) / p.TR;
    if (blockIdx.x >= ntiles) return;
    int64_t nlocal = (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
    uint64_t pol = 0;
    if (p.mode == kModeBulk) {
        pol = policy_evict_first();
        if (threadIdx.x == 0) {
            for (int s = 0; s < p.stages; s++) mbar_init(&mbar[s], 1);
            fence_mbar_init();
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            int64_t pre = nlocal < p.stages ? nlocal : p.stages;
            for (int64_t i = 0; i < pre; i++) stream_issue(p, bufs, mbar, i, pol);
        }
    }
    for (int64_t i = 0; i < nlocal; i++) {
        int s = static_cast<int>(i % p.stages);
        int64_t t = blockIdx.x + i * gridDim.x;
        int64_t r0 = t * p.TR;
        int nr = static_cast<int>(p.R - r0 < p.TR ? p.R - r0 : p.TR);
        unsigned char* buf = bufs + static_cast<size_t>(s) * p.stage_bytes;
        const unsigned char *seg0, *seg1;
        if (p.mode == kModeDirect) {
            seg0 = p.base[0] + r0 * p.rbytes[0];
            seg1 = p.nseg > 1 ? p.base[1] + r0 * p.rbytes[1] : nullptr;
        } else {
            if (p.mode == kModeBulk) {
                mbar_wait(&mbar[s], static_cast<uint32_t>((i / p.stages) & 1));
                if (nr < p.TR) {  // tail tile: sub-16-byte remainder by hand
                    stream_copy_plain(p, buf, r0, nr, true);
                    __syncthreads();
                }
            } else {
                stream_copy_plain(p, buf, r0, nr, false);
                __syncthreads();
            }
            seg0 = buf + p.soff[0];
            seg1 = p.nseg > 1 ? buf + p.soff[1] : nullptr;
        }
        work.tile(seg0, seg1, r0, nr, i);
        // Order this tile's generic-proxy shared-memory traffic before the TMA
        // refill of the same buffer.
        if (p.mode == kModeBulk) fence_proxy_async_smem();
        __syncthreads();
        if (p.mode == kModeBulk && threadIdx.x == 0 && i + p.stages < nlocal)
            stream_issue(p, bufs, mbar, i + p.stages, pol);
        work.finish(r0, nr, i);
    }
}

}  // namespace kr
