// kr_synth.cu -- synthetic trace generation straight into device columns
// (workload.py:296-456 `SyntheticSpec`, `_synth_round_magnitudes`,
// `synthesize_trace`, `synthesize_family`).
//
// The reference draws every round from a sequential numpy Generator per task.
// Bit parity with that generator is not a goal; what is kept is
// the construction: the same distributions, the same per-round magnitude
// formula u[k, n] = u0_n * rho_n^k * noise_kn with the uncertain tail's final
// row set to bump * mean(earlier rows) in numpy's mean order, the horizon of
// each round decided by the policy kernels (bit-exact decide_horizon), and the
// same trigger placement / action-budget loop.  Randomness is counter-based
// (Philox-4x32-10 keyed by (seed, task) and indexed by (round, column,
// purpose)), so a task's rounds do not depend on how many rounds or tasks one
// launch generates.
//
//   k_synth_magnitudes   thread per (task, round, column): K magnitudes + tail
//   k_synth_close        thread per task: consume the decided horizons in order
//                        (trigger placement, executed actions, budget)
//   k_synth_success      thread per task: rng.random() < success_rate
//   k_synth_trajectories thread per (round, dim): cumulative normal steps
#include <cmath>
#include <cstdint>

#include "kr_common.cuh"
#include "kr_host.cuh"

namespace kr {

// Philox-4x32-10 (Salmon et al., SC'11): counter-based, stateless.
struct Philox {
    uint32_t k0, k1;
    __device__ __forceinline__ uint4 operator()(uint4 c) const {
        uint32_t a = k0, b = k1;
#pragma unroll
        for (int r = 0; r < 10; r++) {
            const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
            const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
            c = make_uint4(hi1 ^ c.y ^ a, lo1, hi0 ^ c.w ^ b, lo0);
            a += 0x9E3779B9u;
            b += 0xBB67AE85u;
        }
        return c;
    }
};

__device__ __forceinline__ Philox philox_for(uint64_t seed, int64_t task) {
    // mix the task into the key (splitmix64 finaliser) so tasks are independent streams
    uint64_t z = seed + 0x9E3779B97F4A7C15ull * static_cast<uint64_t>(task + 1);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    return Philox{static_cast<uint32_t>(z), static_cast<uint32_t>(z >> 32)};
}

// [0, 1) with 53 random bits
__device__ __forceinline__ double u01(uint32_t a, uint32_t b) {
    return static_cast<double>((static_cast<uint64_t>(a) << 21) ^ (b >> 11)) * 0x1p-53;
}

// numpy Generator.uniform(lo, hi) = lo + (hi - lo) * U
__device__ __forceinline__ double uniform(double lo, double hi, double u) {
    return dadd(lo, dmul(dadd(hi, -lo), u));
}

enum : uint32_t { kPurposeColumn = 0, kPurposeRound = 1, kPurposeNoise = 2, kPurposeTraj = 3,
                  kPurposeSuccess = 4 };

// workload.py:341-363 `_synth_round_magnitudes`, one (task, round, column)
// per thread.  U is [A][G][K][N] float64.
__global__ void k_synth_magnitudes(kr_synth_spec s, uint64_t seed, const int64_t* __restrict__ tasks,
                                   int64_t A, int32_t round0, int32_t G, double* __restrict__ U) {
    const int K = s.diffusion_steps, N = s.chunk_size;
    const int64_t total = A * G * N;
    const double rlo = fmax(0.05, s.decay - 0.15), rhi = fmin(0.9, s.decay + 0.15);
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int n = static_cast<int>(i % N);
        const int64_t ag = i / N;
        const int g = static_cast<int>(ag % G);
        const int64_t a = ag / G;
        const uint32_t rnd = static_cast<uint32_t>(round0 + g);
        const Philox ph = philox_for(seed, tasks[a]);
        const uint4 c = ph(make_uint4(rnd, static_cast<uint32_t>(n), kPurposeColumn, 0));
        const double rho = uniform(rlo, rhi, u01(c.x, c.y));
        const double u0 = uniform(0.5, 2.0, u01(c.z, c.w));
        // the round's uncertain-tail length: min(1, U(0, 2 f)) * N, rounded half-to-even
        const uint4 cr = ph(make_uint4(rnd, 0, kPurposeRound, 0));
        const double frac = fmin(1.0, uniform(0.0, 2.0 * s.uncertain_fraction, u01(cr.x, cr.y)));
        const int n_unc = static_cast<int>(rint(dmul(frac, static_cast<double>(N))));
        double* col = U + ag * static_cast<int64_t>(K) * N + n;
        double rk = 1.0;  // rho ** k
        for (int k = 0; k < K; k++) {
            const uint4 cn = ph(make_uint4(rnd, static_cast<uint32_t>(n), kPurposeNoise,
                                           static_cast<uint32_t>(k)));
            const double noise = dadd(1.0, uniform(-s.noise_scale, s.noise_scale, u01(cn.x, cn.y)));
            if (k > 0) rk = pow(rho, static_cast<double>(k));
            col[static_cast<int64_t>(k) * N] = dmul(dmul(u0, rk), noise);
        }
        if (n_unc > 0 && n >= N - n_unc) {
            // u[-1, tail] = bump * u[:-1, tail].mean(axis=0): numpy adds the
            // rows in order, except for a single-column tail, whose strided
            // 1-D reduction is numpy's pairwise sum
            double sum;
            if (n_unc == 1) {
                auto at = [col, N](int64_t k) { return col[k * N]; };
                sum = np_pairwise_sum(at, 0, K - 1);
            } else {
                sum = col[0];
                for (int k = 1; k < K - 1; k++) sum = dadd(sum, col[static_cast<int64_t>(k) * N]);
            }
            col[static_cast<int64_t>(K - 1) * N] = dmul(s.bump_factor, ddiv(sum, static_cast<double>(K - 1)));
        }
    }
}

// workload.py:404-436: the rounds of one task in order until the action budget
// is met.  state[a] = {executed, prev_h (-1: none yet), n_rounds, done}.
__global__ void k_synth_close(const int32_t* __restrict__ H, int64_t A, int32_t G, int32_t budget,
                              int32_t slack, int32_t* __restrict__ state,
                              int32_t* __restrict__ trigger, uint8_t* __restrict__ used) {
    for (int64_t a = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; a < A;
         a += int64_t(gridDim.x) * blockDim.x) {
        int32_t* st = state + 4 * a;
        int executed = st[0], prev_h = st[1], nr = st[2], done = st[3];
        for (int g = 0; g < G; g++) {
            const int64_t j = a * G + g;
            if (done) {
                used[j] = 0;
                trigger[j] = 0;
                continue;
            }
            const int h = H[j];
            int t = 0;
            if (prev_h >= 0) {
                t = prev_h - slack;
                t = t < 0 ? 0 : t;
                t = t < prev_h - 1 ? t : prev_h - 1;
            }
            trigger[j] = t;
            used[j] = 1;
            executed += h;
            prev_h = h;
            nr++;
            done = executed >= budget;
        }
        st[0] = executed; st[1] = prev_h; st[2] = nr; st[3] = done;
    }
}

__global__ void k_synth_success(uint64_t seed, const int64_t* __restrict__ tasks, int64_t A,
                                double rate, uint8_t* __restrict__ out) {
    for (int64_t a = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; a < A;
         a += int64_t(gridDim.x) * blockDim.x) {
        const uint4 c = philox_for(seed, tasks[a])(make_uint4(0xFFFFFFFFu, 0, kPurposeSuccess, 0));
        out[a] = u01(c.x, c.y) < rate;
    }
}

// workload.py:417-419: steps = normal(0, 0.05, (h, dim)); cumsum over rows.
// Thread per (round, dim); normals by Box-Muller over two uniforms.
__global__ void k_synth_trajectories(uint64_t seed, const int64_t* __restrict__ task_of,
                                     const int32_t* __restrict__ round_of,
                                     const int32_t* __restrict__ h, const int64_t* __restrict__ row_off,
                                     int64_t nr, int32_t dim, double* __restrict__ traj) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < nr * dim;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = i / dim;
        const int d = static_cast<int>(i % dim);
        const Philox ph = philox_for(seed, task_of[r]);
        double acc = 0.0;
        double* out = traj + row_off[r] * dim + d;
        for (int row = 0; row < h[r]; row++) {
            const uint4 c = ph(make_uint4(static_cast<uint32_t>(round_of[r]), static_cast<uint32_t>(row),
                                          kPurposeTraj, static_cast<uint32_t>(d)));
            const double u1 = 1.0 - u01(c.x, c.y), u2 = u01(c.z, c.w);  // u1 in (0, 1]
            const double z = sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
            acc = dadd(acc, dmul(0.05, z));
            out[static_cast<int64_t>(row) * dim] = acc;
        }
    }
}

static int grid_for(int64_t n, int threads) {
    const int64_t cap = static_cast<int64_t>(device_info().sm_count) * 16;
    int64_t b = (n + threads - 1) / threads;
    return static_cast<int>(b < 1 ? 1 : (b > cap ? cap : b));
}

}  // namespace kr

using namespace kr;

extern "C" int kr_synth_magnitudes(const kr_synth_spec* spec, uint64_t seed, const int64_t* tasks,
                                   int64_t A, int32_t round0, int32_t G, double* U, void* stream) {
    if (!spec || A < 0 || G < 0 || round0 < 0 || spec->chunk_size < 1 || spec->diffusion_steps < 2)
        return KR_EINVAL;
    if (A == 0 || G == 0) return KR_OK;
    if (!tasks || !U) return KR_EINVAL;
    const int64_t n = A * G * spec->chunk_size;
    k_synth_magnitudes<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(*spec, seed, tasks, A, round0,
                                                                         G, U);
    return check_launch("k_synth_magnitudes");
}

extern "C" int kr_synth_close(const int32_t* H, int64_t A, int32_t G, int32_t budget, int32_t slack,
                              int32_t* state, int32_t* trigger, uint8_t* used, void* stream) {
    if (A < 0 || G < 0 || budget < 1 || slack < 0) return KR_EINVAL;
    if (A == 0 || G == 0) return KR_OK;
    if (!H || !state || !trigger || !used) return KR_EINVAL;
    k_synth_close<<<grid_for(A, 128), 128, 0, as_stream(stream)>>>(H, A, G, budget, slack, state, trigger,
                                                                   used);
    return check_launch("k_synth_close");
}

extern "C" int kr_synth_success(uint64_t seed, const int64_t* tasks, int64_t A, double rate,
                                uint8_t* out, void* stream) {
    if (A < 0 || !(rate >= 0.0 && rate <= 1.0)) return KR_EINVAL;
    if (A == 0) return KR_OK;
    if (!tasks || !out) return KR_EINVAL;
    k_synth_success<<<grid_for(A, 128), 128, 0, as_stream(stream)>>>(seed, tasks, A, rate, out);
    return check_launch("k_synth_success");
}

extern "C" int kr_synth_trajectories(uint64_t seed, const int64_t* task_of, const int32_t* round_of,
                                     const int32_t* h, const int64_t* row_off, int64_t nr, int32_t dim,
                                     double* traj, void* stream) {
    if (nr < 0 || dim < 0) return KR_EINVAL;
    if (nr == 0 || dim == 0) return KR_OK;
    if (!task_of || !round_of || !h || !row_off || !traj) return KR_EINVAL;
    k_synth_trajectories<<<grid_for(nr * dim, 128), 128, 0, as_stream(stream)>>>(
        seed, task_of, round_of, h, row_off, nr, dim, traj);
    return check_launch("k_synth_trajectories");
}
