/*
 * kairos_b200.h -- C ABI of the B200-native Kairos decision core.
 *
 * One shared library, libkairos_b200.so (built from
 * paper_2605_11381_b200/csrc/ for sm_100a), exports exactly these entry points.
 * They replace the reference's pure-Python hot path (paths relative to
 * /root/reference/pkg/src/roboserve/):
 *
 *   kr_horizon_confidence   horizon.py:108-132   decide_horizon (confidence branch)
 *   kr_horizon_static       horizon.py:121-122   decide_horizon (static branch)
 *   kr_horizon_sweep        horizon.py:135-151   sweep_thresholds (cli.py:109-140 cmd_pareto)
 *   kr_horizon_divergence   workload.py:461-496  _cosine + round_optimal_horizon
 *   kr_us_from_actions      core.py:24-47,157-166 us_from_actions / exec_end_from_piggyback
 *   kr_wait_ratio           waiting.py:62-66,96-100 wait_ratio / current_wait_ratio
 *   kr_assign_bucket        scheduler.py:79-88   assign_bucket
 *   kr_urgency              waiting.py:69-93 + scheduler.py:79-140,143-157
 *                           ledger, wait ratio, bucket, exec estimate, sort key
 *   kr_topk_select          scheduler.py:204-207 edge prefix S_e = order[:k]
 *   kr_select_admit         scheduler.py:193-241 select + admission + ordered S_e
 *   kr_admit                scheduler.py:223-234 refetch + skip counters
 *   kr_sort_keys            scheduler.py:130-140 the total order itself
 *   kr_merge_runs           sharded admission: W sorted local top-k' lists -> global S_e
 *   kr_ledger_apply         core.py:200-229 + waiting.py:69-93  incremental TaskState
 *                           history and running wait totals (sim.py:358-440 mutations)
 *   kr_urgency_ledger       kr_urgency over the device-resident ledger (O(1) per request)
 *   kr_plan_small           scheduler.py:254-276 plan() edge tier for n <= 4096 in one launch
 *   kr_trace_parse / _load  workload.py:163-262  JSONL task traces -> columns (host code)
 *   kr_transfer_time        engines.py:158-169   per-request uplink time
 *   kr_place_cloud          scheduler.py:160-234 phase-3 cloud offload scan
 *   kr_apply_placements     scheduler.py:223-234 a sharded round's cloud placements on
 *                           their owning shard (skip counter reset, refetch flag)
 *
 * Conventions: every pointer argument that names device data is a device
 * pointer; kr_fleet / kr_sched structs themselves live in host memory.  All
 * calls are asynchronous on `stream` (a cudaStream_t, NULL = legacy default),
 * never allocate, never synchronise (except where documented), and return a
 * kr_status.  Data-dependent validation (non-finite magnitudes, key-field
 * overflow) is reported through a caller-owned device word `flags` that the
 * kernels atomically OR; the host shim raises the reference's ValueError.
 * No C++ exception crosses this boundary.  Stream-ordered and re-entrant per
 * stream; no global mutable state.
 */
#ifndef KAIROS_B200_H
#define KAIROS_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define KR_API __attribute__((visibility("default")))
#else
#define KR_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    KR_OK = 0,
    KR_EINVAL = 1,     /* bad shape / argument (host-side check) */
    KR_ECUDA = 2,      /* CUDA launch / runtime error */
    KR_ENOSPACE = 3,   /* workspace too small */
    KR_EFORMAT = 4,    /* malformed trace file (kr_trace_*: details in the columns' err_*) */
} kr_status;

enum { KR_F32 = 0, KR_F64 = 1 };
enum { KR_KAIROS = 0, KR_FIFO = 1, KR_LAS = 2 };

/* Device validation flags (OR-ed into *flags). */
#define KR_FLAG_NONFINITE  0x1u  /* horizon.py:47-48  "update magnitudes must be finite" */
#define KR_FLAG_NEGATIVE   0x2u  /* horizon.py:49-50  "update magnitudes must be >= 0"   */
#define KR_FLAG_KEY_RANGE  0x4u  /* packed sort-key field out of range */
#define KR_FLAG_TIME_RANGE 0x8u  /* core.py:38-41 negative action count / overflow       */
#define KR_FLAG_RATIO      0x10u /* wait-ratio operand beyond 2^53 (inexact double)      */
#define KR_FLAG_LEDGER     0x20u /* ledger event out of order / beyond capacity        */
#define KR_FLAG_DUP_KEY    0x40u /* sharded merge met one key on two shards (non-global
                                    robot ranks or per-shard issued bases)           */

/* 128-bit composite sort key (ascending = reference order). */
typedef struct kr_key {
    uint64_t hi;
    uint64_t lo;
} kr_key;

/* Fleet structure-of-arrays: one entry per pending request. */
typedef struct kr_fleet {
    int64_t n;
    const int64_t* t_start;          /* TaskState.t_start                     core.py:187 */
    const int64_t* issued_at;        /* PendingRequest.issued_at              core.py:147 */
    const int64_t* obs_captured_at;  /* PendingRequest.obs_captured_at        core.py:148 */
    const int64_t* accum_gen;        /* TaskState.accumulated_generation      core.py:189 */
    const int32_t* remaining;        /* LastExecInfo.remaining_actions        core.py:127 */
    const int32_t* lexrank;          /* position of task_id in sorted(task ids)          */
    int32_t* skipped;                /* PendingRequest.skipped in, TaskState.skipped out  */
    const int64_t* hist_off;         /* CSR slot offset per request                      */
    const int32_t* n_exec;           /* len(TaskState.exec_intervals)                    */
    const int32_t* n_gen;            /* len(TaskState.gen_starts)                        */
    const int64_t* slots;            /* [*][4] gen_start, gen_end, exec_start, exec_end  */
} kr_fleet;

/* Device-resident incremental ledger: per-task state and append-only history
 * (TaskState, core.py:169-249), kept across planning rounds. */
typedef struct kr_ledger {
    int64_t n_tasks;                 /* task slots allocated                            */
    int32_t cap;                     /* history rounds per task                         */
    int32_t pad_;
    int64_t* t_start;                /* [n_tasks] TaskState.t_start                     */
    int32_t* n_exec;                 /* [n_tasks] len(exec_intervals)                   */
    int32_t* n_gen;                  /* [n_tasks] len(gen_starts)                       */
    int32_t* wait_next;              /* [n_tasks] first round whose wait is not final   */
    int64_t* wait_total;             /* [n_tasks] ledger_from_history(state).total_wait */
    int64_t* slots;                  /* [n_tasks][cap][4] gen_start, gen_end (INT64_MIN
                                        while in flight), exec_start, exec_end          */
} kr_ledger;

enum { KR_EV_NEW = 0, KR_EV_BEGIN_GEN = 1, KR_EV_FINISH_GEN = 2, KR_EV_EXEC = 3 };

/* A batch of TaskState mutations grouped by task (each group in call order). */
typedef struct kr_events {
    int64_t n_groups;                /* tasks touched                                   */
    const int32_t* task;             /* [n_groups] task slot                            */
    const int32_t* off;              /* [n_groups + 1] event range of each group        */
    const int32_t* kind;             /* [events] KR_EV_*                                */
    const int32_t* round;            /* [events] round id (unused for KR_EV_NEW)        */
    const int64_t* a;                /* [events] t_start / at / at / exec start         */
    const int64_t* b;                /* [events] exec end (KR_EV_EXEC)                  */
} kr_events;

/* One planning round's pending requests against a kr_ledger. */
typedef struct kr_requests {
    int64_t n;
    const int32_t* task;             /* task slot of each request                       */
    const int64_t* issued_at;
    const int64_t* obs_captured_at;
    const int64_t* accum_gen;        /* TaskState.accumulated_generation (LAS key)      */
    const int32_t* remaining;
    const int32_t* lexrank;
    int32_t* skipped;                /* PendingRequest.skipped in, updated by admission */
} kr_requests;

/* SchedulerConfig (scheduler.py:38-56) plus the round's scalars. */
typedef struct kr_sched {
    int32_t policy;                  /* KR_KAIROS / KR_FIFO / KR_LAS */
    int32_t buckets;                 /* B, 1..256 */
    int32_t aging_interval;          /* A >= 1 */
    int32_t pad_;
    int64_t stale_threshold;         /* µs */
    int64_t default_exec_estimate;   /* µs */
    int64_t now;                     /* µs */
    int64_t hz_num, hz_den;          /* control_hz == hz_num / hz_den exactly */
    int64_t issued_base;             /* key origin: issued_at - issued_base in [0, 2^40) */
} kr_sched;

KR_API const char* kr_version(void);
KR_API const char* kr_status_string(int status);
/* Last CUDA error string recorded by a failing call on this thread. */
KR_API const char* kr_last_error(void);
/* Kernels launched by this library so far in this process (diagnostic). */
KR_API unsigned long long kr_launch_count(void);
/* Stream-ordered copy between any two addresses (cudaMemcpyDefault): stages a
 * scalar call's inputs from the mapped arena into device scratch. */
KR_API int kr_memcpy_async(void* dst, const void* src, size_t bytes, void* stream);
/* cudaStreamSynchronize(stream): the one wait of a small synchronous call. */
KR_API int kr_stream_synchronize(void* stream);

/* ---- step 1: execution-horizon selection ------------------------------ */

/* U: [R][K][N] fp32 (dtype KR_F32) or fp64, row-major.  H[r] = decide_horizon.
 * one_plus_t = 1.0 + threshold computed on the host in fp64 (horizon.py:127).
 * max_sms (0 = all) caps the persistent grid as for kr_horizon_divergence. */
KR_API int kr_horizon_confidence(const void* U, int dtype, int64_t R, int32_t K, int32_t N,
                          double one_plus_t, int32_t min_horizon, int32_t* H,
                          uint32_t* flags, int32_t max_sms, void* stream);
KR_API int kr_horizon_static(int64_t R, int32_t N, int32_t static_h, int32_t* H, void* stream);

/* C <= 64 policy configurations decided over the same rounds U[R][K][N] in
 * one pass (sweep_thresholds / cmd_pareto).  Host arrays per configuration:
 * kind[c] 0 = static (param[c] = static_h), 1 = confidence (one_plus_t[c] =
 * 1.0 + threshold, param[c] = min_horizon).  sums[c] (device, caller-zeroed,
 * accumulated) += sum_r decide_horizon(cfg_c, U[r]); H (nullable) [C][R]
 * receives every decision.  The reference's mean is sums[c] / R. */
KR_API int kr_horizon_sweep(const void* U, int dtype, int64_t R, int32_t K, int32_t N, int32_t C,
                            const int32_t* kind, const double* one_plus_t, const int32_t* param,
                            unsigned long long* sums, int32_t* H, uint32_t* flags, void* stream);

/* prev: [R][Lp][D], cand: [R][S][Lc][D] (same dtype).  For robot r the
 * reference trajectory is prev[r][off_r : len_prev_r] (the unexecuted overlap
 * of the previous chunk), the candidates cand[r][s][0 : len_cand_r].
 * H[r] = min_s round_optimal_horizon(ref_r, cand_{r,s}, thr).  offset /
 * len_prev / len_cand may be NULL (0 / Lp / Lc).  cos (nullable) receives the
 * fp64 cosine of every (r, s, i < limit_r), NaN beyond the limit. */
/* Exact-cosine ddot order (workload.py:461-468 `_cosine` through numpy's
 * OpenBLAS): the reference's fp64 cosines are those of the BLAS core numpy
 * selected at run time, so the order is a process-wide setting that the host
 * takes from threadpoolctl's report (OpenBLAS 0.3.30 cores SkylakeX /
 * Cooperlake / SapphireRapids -> KR_DOT_SKYLAKEX, Haswell / Zen ->
 * KR_DOT_HASWELL).  Read when a launch is set up.  Default KR_DOT_SKYLAKEX. */
#define KR_DOT_SKYLAKEX 0
#define KR_DOT_HASWELL  1
KR_API int kr_set_dot_order(int32_t order);
KR_API int32_t kr_get_dot_order(void);

KR_API int kr_horizon_divergence(const void* prev, const void* cand, int dtype, int64_t R,
                          int32_t S, int32_t Lp, int32_t Lc, int32_t D,
                          const int32_t* offset, const int32_t* len_prev,
                          const int32_t* len_cand, double thr, int32_t* H, double* cos,
                          int32_t max_sms, void* stream);
/* max_sms (0 = all): cap the persistent grid to this many SMs so that work on
 * another stream (urgency + admission, which do not depend on H) can run on
 * the remaining SMs concurrently. */

/* ---- step 2: execution-aware urgency ---------------------------------- */

/* out[i] = (base ? base[i] : 0) + us_from_actions(count[i], hz_num/hz_den). */
KR_API int kr_us_from_actions(const int64_t* count, const int64_t* base, int64_t n, int64_t hz_num,
                       int64_t hz_den, int64_t* out, uint32_t* flags, void* stream);
/* wr[i] = current_wait_ratio semantics: 0 if now <= t_start[i]. */
KR_API int kr_wait_ratio(const int64_t* total_wait, const int64_t* t_start, int64_t n, int64_t now,
                  double* wr, uint32_t* flags, void* stream);
KR_API int kr_assign_bucket(const double* wr, const int32_t* skipped, int64_t n, int32_t buckets,
                     int32_t aging_interval, int32_t* bucket, void* stream);
/* Fused per-request pass: ledger -> wait ratio -> bucket -> exec estimate ->
 * aged estimate -> packed key (+ next-need time).  Optional outputs nullable;
 * slot_wait[hist_off + j] receives round j's recorded wait, or -1 where the
 * ledger records none (WaitLedger.waits, waiting.py:82-92). */
KR_API int kr_urgency(const kr_fleet* fleet, const kr_sched* cfg, kr_key* keys, int64_t* need_time,
               int64_t* total_wait, double* wr, int32_t* bucket, int64_t* est,
               int64_t* slot_wait, unsigned long long* key_stats, uint32_t* flags, void* stream);
/* The planning round's urgency pass (kr_urgency with keys and need times)
 * whose last CTA also prepares the radix-select state in `workspace` for
 * kr_select_admit_prepared with budget k: the state reset and level-0 digit
 * of kr_select_admit's first launch, from the keys' statistics this pass
 * reduces (per-CTA partials in the workspace, no key_stats buffer, no
 * kr_key_stats_init).  workspace as for kr_select_admit over fleet->n keys;
 * fleet->n >= 16,384 (smaller rounds sort every key instead), and its state's
 * completion counter zero before the first call (a zeroed workspace).
 * scheduler.py:120-140 (keys) + the select preparation; waiting.py:69-100. */
KR_API int kr_urgency_prep(const kr_fleet* fleet, const kr_sched* cfg, kr_key* keys,
                           int64_t* need_time, uint32_t* flags, int64_t k, void* workspace,
                           size_t workspace_bytes, void* stream);
/* key_stats (nullable, 4 words, prepared by kr_key_stats_init) accumulates
 * {OR hi, OR lo, AND hi, AND lo} of the keys written, so the admission select
 * needs no extra pass over the keys. */
KR_API int kr_key_stats_init(unsigned long long* key_stats, void* stream);

/* A whole edge-tier planning round for n <= 4096 pending requests in ONE
 * launch (replaces plan(), scheduler.py:254-276, at the simulator's call
 * sizes: sim.py:298-308): urgency keys, the total order (one-CTA bitonic
 * sort), admission of the first min(k, n), stale-observation refetch and the
 * skip counter update.  The fleet columns may point to mapped pinned host
 * memory (kr_mapped_ptr) and so may `out`; out = int32 [3n + 1]: order[n]
 * (request indices, plan order), refetch[n] and updated skipped[n] (both by
 * request index), then the validation flags word.  fleet->skipped is NOT
 * modified.  KR_EINVAL for n > 4096. */
KR_API int kr_plan_small(const kr_fleet* fleet, const kr_sched* cfg, int64_t k, int32_t* out,
                         void* stream);
/* Device address of mapped pinned host memory (cudaHostGetDevicePointer). */
KR_API int kr_mapped_ptr(void* host, void** device);

/* Apply a batch of TaskState mutations to the device ledger (one thread per
 * task; wait totals advance incrementally).  Out-of-order rounds or rounds
 * beyond ledger->cap set KR_FLAG_LEDGER and are skipped. */
KR_API int kr_ledger_apply(const kr_ledger* ledger, const kr_events* events, uint32_t* flags,
                           void* stream);
/* kr_urgency over ledger-backed requests: identical keys / outputs, with the
 * total wait and last execution read in O(1) per request. */
KR_API int kr_urgency_ledger(const kr_ledger* ledger, const kr_requests* req, const kr_sched* cfg,
                             kr_key* keys, int64_t* need_time, int64_t* total_wait, double* wr,
                             int32_t* bucket, int64_t* est, unsigned long long* key_stats,
                             uint32_t* flags, void* stream);

/* ---- step 3: priority ordering + top-k admission ---------------------- */

/* Bytes of scratch needed by kr_topk_select / kr_sort_keys for n keys. */
KR_API size_t kr_workspace_bytes(int64_t n);
/* Device-side k-th smallest key (MSD radix select).  *kth is undefined for
 * k == 0; for k >= n it is the all-ones key. */
KR_API int kr_topk_select(const kr_key* keys, int64_t n, int64_t k, kr_key* kth,
                          const unsigned long long* key_stats, void* workspace,
                          size_t workspace_bytes, void* stream);
/* Admission pass over n keys (scheduler.py:204-207, 223-234):
 *   admitted[i] = k > 0 && (kth == NULL || key_i <= *kth)
 * (kth NULL with k > 0 admits everything, i.e. k >= n), refetch[i] = admitted
 * && now - obs_captured_at > stale_threshold, skip counters updated in place
 * (admitted -> 0, deferred -> skipped + 1).  With edge_idx / edge_keys the
 * admitted (key, index) pairs -- exactly min(k, n) of them when kth is the
 * k-th smallest key -- are gathered and sorted, so edge_idx is S_e in
 * reference order.  admitted / refetch / edge outputs nullable; fleet / cfg
 * may be NULL when neither refetch nor skip counters are wanted. */
KR_API int kr_admit(const kr_key* keys, int64_t n, int64_t k, const kr_key* kth,
             const kr_fleet* fleet, const kr_sched* cfg, uint8_t* admitted, uint8_t* refetch,
             int32_t* edge_idx, kr_key* edge_keys, void* workspace, size_t workspace_bytes,
             void* stream);
/* Fused top-k admission (the production path): select the k-th key, admit
 * key <= kth with masks / refetch / skip counters, and write S_e ordered into
 * edge_idx / edge_keys (the admitted keys are gathered straight into the
 * select's level-0 bin order and each bin is sorted in shared memory).
 * kth_out (nullable) receives the k-th key.  key_stats as for kr_topk_select. */
KR_API int kr_select_admit(const kr_key* keys, int64_t n, int64_t k,
                           const unsigned long long* key_stats, const kr_fleet* fleet,
                           const kr_sched* cfg, uint8_t* admitted, uint8_t* refetch,
                           int32_t* edge_idx, kr_key* edge_keys, kr_key* kth_out, void* workspace,
                           size_t workspace_bytes, void* stream);
/* kr_select_admit after kr_urgency_prep prepared the select state in the same
 * workspace for the same keys and k (no state-reset launch, no statistics
 * argument).  Identical outputs. */
KR_API int kr_select_admit_prepared(const kr_key* keys, int64_t n, int64_t k,
                                    const kr_fleet* fleet, const kr_sched* cfg, uint8_t* admitted,
                                    uint8_t* refetch, int32_t* edge_idx, kr_key* edge_keys,
                                    kr_key* kth_out, void* workspace, size_t workspace_bytes,
                                    void* stream);
/* Sharded admission (rounds.sharded_topk): `runs` holds W ascending runs of
 * `len` keys each (every rank's local top-k' candidates, all-ones padded, as
 * all-gathered).  Writes the k smallest keys overall, in order, to out_keys
 * (nullable) and the k-th smallest to kth_out (nullable); k <= W * len.
 * The merge is exact for unique keys only: a non-padding key that occurs
 * twice sets KR_FLAG_DUP_KEY in *flags (nullable). */
KR_API int kr_merge_runs(const kr_key* runs, int32_t W, int64_t len, int64_t k, kr_key* out_keys,
                         kr_key* kth_out, uint32_t* flags, void* stream);
/* kr_merge_runs that also records, for each output rank, the element's
 * position in `runs` (run r, slot j -> r * len + j): lets a caller carry
 * per-candidate payloads (e.g. uplink times for the cloud scan) through the
 * merge.  out_pos may be NULL. */
KR_API int kr_merge_runs_pos(const kr_key* runs, int32_t W, int64_t len, int64_t k,
                             kr_key* out_keys, int32_t* out_pos, kr_key* kth_out, uint32_t* flags,
                             void* stream);

/* ---- phase 3: hybrid edge / cloud placement --------------------------- */

/* out[i] = base_us + round_half_up(payload[i] * 8e6 / bps)   (engines.py:158-169) */
KR_API int kr_transfer_time(const int64_t* payload, int64_t n, int64_t base_us, int64_t bps,
                            int64_t* out, void* stream);
/* scheduler.py:210-234 cloud offload after the edge prefix of `order` (the
 * full reference order, n_edge = |S_e|): request r is offloaded iff
 * up_us[r] < thresholds[c] with c = offloads so far (< cap), where
 * thresholds[c] = edge_est - (cloud drain(c) + cloud batch latency(c) +
 * downlink), INT64_MAX without an edge tier.  Offloaded requests get skip
 * counter 0 and their refetch flag; cloud_idx[0..*n_cloud) is S_c in order. */
KR_API int kr_place_cloud(const int32_t* order, int64_t n, int64_t n_edge, const int64_t* up_us,
                          const int64_t* thresholds, int64_t cap, const kr_fleet* fleet,
                          const kr_sched* cfg, uint8_t* refetch, int32_t* cloud_idx,
                          int32_t* n_cloud, void* stream);

/* scheduler.py:223-234 for a robot-sharded round's offload set: pos[i] for
 * i < *n_placed (device count, e.g. kr_place_cloud's n_cloud) are positions in
 * the all-gathered candidate runs of length run_len; those in run `rank` (this
 * shard) name local robot cand_idx[pos % run_len], whose skip counter is reset
 * and refetch flag set (now - obs_captured_at > stale_threshold).  No host
 * synchronisation: the count stays on the device. */
KR_API int kr_apply_placements(const int32_t* pos, const int32_t* n_placed, int64_t cap,
                               int64_t run_len, int32_t rank, const int32_t* cand_idx,
                               const kr_fleet* fleet, const kr_sched* cfg, uint8_t* refetch,
                               void* stream);

/* ---- trace ingest (host code): JSON Lines task traces -> columns -------- */

/* Columnar view of a parsed trace file (workload.py:60-262 TaskTrace /
 * RoundRecord).  All pointers are host memory owned by the table. */
typedef struct kr_trace_columns {
    int64_t n_traces, n_rounds, n_mag_values, n_traj_rows, n_traj_values;
    const int64_t* round_off;            /* [n_traces + 1] rounds of trace i            */
    const char* ids;                     /* task ids, UTF-8, concatenated               */
    const int64_t* id_off;               /* [n_traces + 1]                               */
    const double* control_hz;            /* [n_traces]                                   */
    const uint8_t* control_hz_is_int;    /* [n_traces] the JSON literal was an integer   */
    const int64_t* obs_payload_bytes;    /* [n_traces]                                   */
    const int64_t* action_payload_bytes; /* [n_traces]                                   */
    const uint8_t* success;              /* [n_traces] bool(value)                       */
    const int32_t* round_id;             /* [n_rounds]                                   */
    const int32_t* trigger_action_index; /* [n_rounds]                                   */
    const int32_t* horizon;              /* [n_rounds]                                   */
    const int32_t* chunk_size;           /* [n_rounds]                                   */
    const int32_t* mag_k;                /* [n_rounds] K of update_magnitudes (0: none)  */
    const int32_t* mag_n;                /* [n_rounds] N                                 */
    const int64_t* mag_off;              /* [n_rounds + 1] offsets into mags (values)    */
    const double* mags;                  /* K x N row-major per round, concatenated      */
    const int32_t* traj_rows;            /* [n_rounds] rows of action_trajectory (-1: none) */
    const int64_t* traj_row0;            /* [n_rounds + 1] first row of each round       */
    const int64_t* traj_off;             /* [n_traj_rows + 1] offsets into traj (values) */
    const double* traj;
    /* KR_EFORMAT: TraceFormatError fields (workload.py:29-54) */
    int64_t err_line;
    int32_t err_has_task, err_has_round;
    const char* err_task;
    int64_t err_round;
    const char* err_message;
} kr_trace_columns;

/* Parse JSON Lines (load_traces semantics: stripped lines, blanks skipped,
 * the reference's validation order and messages).  *table is always set
 * (free it with kr_trace_free); KR_EFORMAT leaves the traces before the bad
 * line in the columns and the error in err_*. */
KR_API int kr_trace_parse(const char* buf, size_t len, int64_t first_line, void** table);
KR_API int kr_trace_load(const char* path, void** table);
KR_API const kr_trace_columns* kr_trace_columns_of(const void* table);
KR_API void kr_trace_free(void* table);

/* Full argsort of n unique keys (ascending).  Synchronises `stream` once
 * when n exceeds the single-CTA limit (pass plan read back to the host). */
KR_API int kr_sort_keys(const kr_key* keys, int64_t n, int32_t* order, kr_key* sorted_keys,
                 void* workspace, size_t workspace_bytes, void* stream);


/* ---- synthetic traces (workload.py:296-456) -------------------
 * The reference's construction on the device with counter-based randomness
 * (Philox-4x32-10 keyed by (seed, task id), indexed by (round, column)); bit
 * parity with numpy's Generator is not a goal.  `SyntheticSpec` fields that the
 * kernels read: */
typedef struct kr_synth_spec {
    int32_t chunk_size;        /* N */
    int32_t diffusion_steps;   /* K */
    double decay, noise_scale, bump_factor, uncertain_fraction;
} kr_synth_spec;
/* workload.py:341-363 `_synth_round_magnitudes` for rounds [round0, round0+G)
 * of the tasks tasks[A] (any int64 ids) -> U[A][G][K][N] float64 (device). */
KR_API int kr_synth_magnitudes(const kr_synth_spec* spec, uint64_t seed, const int64_t* tasks,
                               int64_t A, int32_t round0, int32_t G, double* U, void* stream);
/* workload.py:404-436: consume the decided horizons H[A][G] of each task in
 * order: trigger placement (max(0, prev_h - slack), at most prev_h - 1), the
 * executed-action total and the budget.  state[A][4] = {executed, prev_h (-1:
 * none), n_rounds, done}, carried across calls; trigger[A][G]; used[A][G]. */
KR_API int kr_synth_close(const int32_t* H, int64_t A, int32_t G, int32_t budget, int32_t slack,
                          int32_t* state, int32_t* trigger, uint8_t* used, void* stream);
/* workload.py:438: success = rng.random() < success_rate, per task. */
KR_API int kr_synth_success(uint64_t seed, const int64_t* tasks, int64_t A, double rate,
                            uint8_t* success, void* stream);
/* workload.py:417-419: per round r, h[r] rows x dim cumulative sums of
 * normal(0, 0.05) steps into traj[row_off[r] + row][dim]. */
KR_API int kr_synth_trajectories(uint64_t seed, const int64_t* task_of, const int32_t* round_of,
                                 const int32_t* h, const int64_t* row_off, int64_t nr, int32_t dim,
                                 double* traj, void* stream);

#ifdef __cplusplus
}
#endif
#endif
