// kr_sweep_f32.cu -- the float instantiation of the threshold-sweep launcher.
#include "kr_sweep.cuh"

namespace kr {
int sweep_run_f32(const void* U, int64_t R, int32_t K, int32_t N, int32_t C, int32_t Cc,
                  const SweepCfg& cfg, unsigned long long* sums, int32_t* H, uint32_t* flags,
                  cudaStream_t st, int max_sms) {
    return sweep_run<float>(U, R, K, N, C, Cc, cfg, sums, H, flags, st, max_sms);
}
}  // namespace kr
