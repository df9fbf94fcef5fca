// kr_host.cuh -- host-side helpers shared by the C-ABI translation units:
// error capture (no exceptions cross the ABI), device properties and the
// launch-shape policy for the persistent streaming kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "../../include/kairos_b200.h"

namespace kr {

void set_last_error(const char* where, cudaError_t e);

// Process-wide count of kernels launched by this library (diagnostic only).
void count_launches(int n);

inline int check_launch(const char* where, int launches = 1) {
    count_launches(launches);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_last_error(where, e);
        return KR_ECUDA;
    }
    return KR_OK;
}

// Programmatic dependent launch for the admission chain's kernels (each
// begins with griddep_wait(), so it may be scheduled while its same-stream
// predecessor drains and then waits for that grid's completion and memory
// flush): the launch latency of one kernel overlaps the tail of the previous.
// KR_NO_PDL=1 launches them plainly (A/B knob).  A failed launch leaves its
// error for check_launch, like <<<>>>.
inline bool pdl_on() {
    static const bool off = std::getenv("KR_NO_PDL") != nullptr;
    return !off;
}
template <typename... ExpTypes, typename... ActTypes>
inline void launch_pdl(void (*kern)(ExpTypes...), dim3 grid, dim3 block, cudaStream_t st,
                       ActTypes&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl_on() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    (void)cudaLaunchKernelEx(&cfg, kern, static_cast<ExpTypes>(args)...);
}

#define KR_CUDA_TRY(expr)                                  \
    do {                                                   \
        cudaError_t kr_e_ = (expr);                        \
        if (kr_e_ != cudaSuccess) {                        \
            ::kr::set_last_error(#expr, kr_e_);            \
            return KR_ECUDA;                               \
        }                                                  \
    } while (0)

struct DeviceInfo {
    int device = -1;
    int sm_count = 0;
    int max_smem_optin = 0;
};
// Properties of the current device (cached per device id).
const DeviceInfo& device_info();

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Resident CTAs per SM of `kernel` at `threads` (>= 1).
template <class K>
inline int occupancy(K kernel, int threads, size_t smem = 0) {
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, threads, smem) != cudaSuccess)
        b = 1;
    return b < 1 ? 1 : b;
}
// CTAs covering n items at `threads` per CTA, capped at one resident wave.
inline unsigned grid_cap(int64_t n, int threads, int per_sm) {
    int64_t b = (n + threads - 1) / threads;
    const int64_t cap = static_cast<int64_t>(device_info().sm_count) * per_sm;
    if (b > cap) b = cap;
    return static_cast<unsigned>(b < 1 ? 1 : b);
}

}  // namespace kr
