/*
 * kairos_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C CPU restatement of the Kairos decision core as implemented by the
 * reference package `roboserve` (/root/reference/pkg/src/roboserve).  It is the
 * parity checker for the CUDA library and the CPU baseline timed by bench.py;
 * it is never linked into, loaded by, or called from the product path
 * (paper_2605_11381_b200/).  Only tests/, __graft_entry__.smoke() and bench.py
 * (cpu_baseline leg and --impl reference) may use it.
 *
 * Parity pinning: tests/golden/ holds vectors produced by running the
 * reference itself in the build container (tests/golden/make_golden.py);
 * tests/test_oracle_golden.py checks this restatement against every one of
 * them plus the reference test-suite's hand-written goldens.
 *
 * Floating-point order: every fp64 operation is written out explicitly and the
 * file is compiled with -ffp-contract=off; fma() appears exactly where the
 * reference's numpy / OpenBLAS 0.3.30 (SkylakeX core) code path fuses.
 */
#ifndef KAIROS_ORACLE_H
#define KAIROS_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* numpy 2.3 `u[:-1].mean(axis=0)` element n of a row-major [rows, N] block. */
double orc_np_mean_col(const double* u, int64_t rows, int64_t N, int64_t n);
/* OpenBLAS 0.3.30 ddot, contiguous, in the order of the BLAS core selected
 * with orc_set_dot_order (process-wide, like OpenBLAS' own core choice):
 * ORC_DOT_SKYLAKEX (default; SkylakeX / Cooperlake / SapphireRapids cores) or
 * ORC_DOT_HASWELL (Haswell / Zen cores). */
#define ORC_DOT_SKYLAKEX 0
#define ORC_DOT_HASWELL 1
int orc_set_dot_order(int order);
int orc_get_dot_order(void);
double orc_ddot(const double* x, const double* y, int64_t n);
/* workload.py:461-468 `_cosine(a, b)`. */
double orc_cosine(const double* a, const double* b, int64_t D);

/* horizon.py:108-132 decide_horizon, confidence branch on one fp64 [K,N]. */
int32_t orc_decide_horizon_conf(const double* u, int64_t K, int64_t N,
                                double one_plus_t, int64_t min_horizon);
/* workload.py:471-496 round_optimal_horizon on fp64 [Lr,D] and [Lc,D]. */
int64_t orc_round_optimal_horizon(const double* ref, int64_t Lr,
                                  const double* cand, int64_t Lc, int64_t D,
                                  double thr);

/* Batched forms over fleet-major tensors (fp32 storage when is_f64 == 0;
 * values are upcast exactly, as np.asarray(float32 -> float64) does). */
void orc_horizon_conf_batch(const void* U, int is_f64, int64_t R, int64_t K,
                            int64_t N, double one_plus_t, int64_t min_horizon,
                            int32_t* H, int nthreads);
/* prev [R,Lp,D], cand [R,S,Lc,D].  Reference rows of robot r are
 * prev[r, off_r : len_prev_r], candidate rows cand[r, s, : len_cand_r]
 * (offset/len arrays may be NULL: 0 / Lp / Lc).  H[r] = min over s of
 * round_optimal_horizon(ref_r, cand_{r,s}, thr).  cos (nullable) receives
 * every cosine [R,S,Lc] up to the limit (NaN past it). */
void orc_divergence_batch(const void* prev, const void* cand, int is_f64,
                          int64_t R, int64_t S, int64_t Lp, int64_t Lc,
                          int64_t D, const int32_t* offset,
                          const int32_t* len_prev, const int32_t* len_cand,
                          double thr, int32_t* H, double* cos, int nthreads);

/* core.py:24-47 us_from_actions with control_hz == hz_num / hz_den exactly. */
int64_t orc_us_from_actions(int64_t count, int64_t hz_num, int64_t hz_den);
/* waiting.py:69-93 ledger_from_history(...).total_wait over CSR slots
 * (gen_start, gen_end, exec_start, exec_end) per round. */
int64_t orc_total_wait(const int64_t* slots, int32_t n_exec, int32_t n_gen);
/* waiting.py:96-100 current_wait_ratio. */
double orc_current_wait_ratio(int64_t total_wait, int64_t t_start, int64_t now);
/* scheduler.py:79-88 assign_bucket. */
int32_t orc_assign_bucket(double wr, int64_t skipped, int64_t buckets,
                          int64_t aging_interval);

/* Fleet structure-of-arrays, one entry per pending request. */
typedef struct {
    int64_t n;
    const int64_t* t_start;          /* TaskState.t_start */
    const int64_t* issued_at;        /* PendingRequest.issued_at */
    const int64_t* obs_captured_at;  /* PendingRequest.obs_captured_at */
    const int64_t* accum_gen;        /* TaskState.accumulated_generation */
    const int32_t* remaining;        /* last_exec_info.remaining_actions */
    const int32_t* lexrank;          /* rank of task_id in sorted(ids) */
    const int32_t* skipped;          /* PendingRequest.skipped */
    const int64_t* hist_off;         /* CSR offset (in slots) */
    const int32_t* n_exec;           /* len(exec_intervals) */
    const int32_t* n_gen;            /* len(gen_starts) */
    const int64_t* slots;            /* [*,4] gen_start gen_end exec_start exec_end */
} orc_fleet;

enum { ORC_KAIROS = 0, ORC_FIFO = 1, ORC_LAS = 2 };

/* scheduler.py:254-276 plan() restricted to the edge tier (no cloud):
 * order[n] = reference order (edge prefix then deferred), per-request
 * intermediates (nullable), admitted/refetch masks and new skip counters.
 * Returns the number admitted to the edge. */
int64_t orc_plan(const orc_fleet* f, int policy, int64_t buckets,
                 int64_t aging_interval, int64_t stale_threshold,
                 int64_t default_exec_estimate, int64_t now, int64_t hz_num,
                 int64_t hz_den, int64_t edge_avail, int32_t* order,
                 int64_t* total_wait, double* wr, int32_t* bucket,
                 int64_t* est, int64_t* need_time, uint8_t* admitted,
                 uint8_t* refetch, int32_t* skipped_out);

/* ---- phase 3: hybrid edge / cloud placement (scheduler.py:160-241) ---- */
typedef struct {
    int64_t capacity, max_batch;
    int32_t npts;
    const int64_t* batch;    /* profiled batch sizes, increasing */
    const int64_t* latency;  /* µs, non-decreasing */
} orc_profile;
typedef struct {
    int64_t base_latency_us, uplink_bps, downlink_bps;
} orc_net;

/* engines.py:132-155 */
int64_t orc_batch_latency(const orc_profile* p, int64_t batch);
/* engines.py:158-169 (up != 0: uplink) */
int64_t orc_transfer_time(const orc_net* net, int64_t payload_bytes, int up);

/* plan() with optional edge / cloud profiles and network model.  tier[i]:
 * 0 deferred, 1 edge, 2 cloud; cloud_order receives the S_c indices in
 * order; returns the number placed on the cloud (edge count via *n_edge). */
int64_t orc_plan_tiers(const orc_fleet* f, const int64_t* payload, int policy, int64_t buckets,
                       int64_t aging_interval, int64_t stale_threshold,
                       int64_t default_exec_estimate, int64_t now, const orc_profile* edge,
                       const orc_profile* cloud, const orc_net* net, int64_t edge_in_flight,
                       int64_t cloud_in_flight, int32_t* order, uint8_t* tier,
                       int32_t* cloud_order, uint8_t* refetch, int32_t* skipped_out,
                       int64_t* n_edge);

#ifdef __cplusplus
}
#endif
#endif
