// kr_sweep_f64.cu -- the double instantiation of the threshold-sweep launcher.
#include "kr_sweep.cuh"

namespace kr {
int sweep_run_f64(const void* U, int64_t R, int32_t K, int32_t N, int32_t C, int32_t Cc,
                  const SweepCfg& cfg, unsigned long long* sums, int32_t* H, uint32_t* flags,
                  cudaStream_t st, int max_sms) {
    return sweep_run<double>(U, R, K, N, C, Cc, cfg, sums, H, flags, st, max_sms);
}
}  // namespace kr
