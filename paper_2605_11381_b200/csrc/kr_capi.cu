// kr_capi.cu -- library-wide C-ABI entry points: version, status strings,
// per-thread last-error capture and the cached device properties used by the
// launch planners.
#include <atomic>
#include <cstdio>
#include <mutex>

#include "kr_host.cuh"

namespace kr {

static thread_local char g_last_error[512] = "";
static std::atomic<unsigned long long> g_launches{0};

void count_launches(int n) { g_launches.fetch_add(static_cast<unsigned long long>(n)); }

void set_last_error(const char* where, cudaError_t e) {
    std::snprintf(g_last_error, sizeof(g_last_error), "%s: %s (%s)", where, cudaGetErrorString(e),
                  cudaGetErrorName(e));
}

const DeviceInfo& device_info() {
    static DeviceInfo cache[64];
    static std::mutex mu;
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    DeviceInfo& d = cache[dev];
    if (d.device != dev) {
        std::lock_guard<std::mutex> lock(mu);
        if (d.device != dev) {
            cudaDeviceGetAttribute(&d.sm_count, cudaDevAttrMultiProcessorCount, dev);
            cudaDeviceGetAttribute(&d.max_smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
            if (d.sm_count <= 0) d.sm_count = 148;
            if (d.max_smem_optin <= 0) d.max_smem_optin = 227 * 1024;
            d.device = dev;
        }
    }
    return d;
}

}  // namespace kr

extern "C" const char* kr_version(void) {
    return "kairos_b200 0.1.0 (sm_100a; fp64 reference-order numerics; OpenBLAS SkylakeX ddot)";
}

extern "C" const char* kr_status_string(int status) {
    switch (status) {
        case KR_OK: return "ok";
        case KR_EINVAL: return "invalid argument";
        case KR_ECUDA: return "CUDA error";
        case KR_ENOSPACE: return "workspace too small";
        case KR_EFORMAT: return "malformed trace data";
        default: return "unknown status";
    }
}

extern "C" const char* kr_last_error(void) { return kr::g_last_error; }

extern "C" unsigned long long kr_launch_count(void) { return kr::g_launches.load(); }

extern "C" int kr_stream_synchronize(void* stream) {
    KR_CUDA_TRY(cudaStreamSynchronize(kr::as_stream(stream)));
    return KR_OK;
}

extern "C" int kr_memcpy_async(void* dst, const void* src, size_t bytes, void* stream) {
    if ((!dst || !src) && bytes) return KR_EINVAL;
    if (bytes == 0) return KR_OK;
    KR_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, kr::as_stream(stream)));
    return KR_OK;
}
