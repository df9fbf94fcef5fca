/*
 * kairos_oracle.c -- TEST INFRASTRUCTURE ONLY (see kairos_oracle.h).
 *
 * CPU restatement of the reference's hot path, one function per reference
 * function, each citing the file:line it follows (paths relative to
 * /root/reference/pkg/src/roboserve/).  Compiled with -ffp-contract=off so the
 * compiler never fuses; fma() is written where numpy/OpenBLAS fuse.
 */
#include "kairos_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

/* ---------------------------------------------------------------------------
 * numpy reductions
 * ------------------------------------------------------------------------- */

/* numpy/_core/src/umath/loops_utils.h.src DOUBLE_pairwise_sum (numpy 2.3):
 * < 8 elements sequential from 0.0; <= 128 eight accumulators; else recurse
 * on halves split at a multiple of 8. */
static double np_pairwise_sum(const double* a, int64_t n, int64_t stride) {
    if (n < 8) {
        double res = 0.0;
        for (int64_t i = 0; i < n; i++) res += a[i * stride];
        return res;
    } else if (n <= 128) {
        double r[8];
        int64_t i;
        for (int j = 0; j < 8; j++) r[j] = a[j * stride];
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; j++) r[j] += a[(i + j) * stride];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++) res += a[i * stride];
        return res;
    } else {
        int64_t n2 = n / 2;
        n2 -= n2 % 8;
        return np_pairwise_sum(a, n2, stride) +
               np_pairwise_sum(a + n2 * stride, n - n2, stride);
    }
}

/* horizon.py:125 `u[:-1].mean(axis=0)`: for N >= 2 the reduction's inner
 * loop runs along N, so each column is a sequential add over rows starting
 * from row 0; for N == 1 the iterator collapses to one contiguous reduce and
 * numpy uses pairwise summation.  Then true-divide by the row count. */
double orc_np_mean_col(const double* u, int64_t rows, int64_t N, int64_t n) {
    double s;
    if (N == 1) {
        s = np_pairwise_sum(u, rows, 1);
    } else {
        s = u[n];
        for (int64_t k = 1; k < rows; k++) s = s + u[k * N + n];
    }
    return s / (double)rows;
}

/* OpenBLAS 0.3.30 kernel/x86_64/ddot.c + ddot_microk_skylakex-2.c (the
 * runtime core numpy's bundled scipy-openblas selects on this host, as
 * recorded by threadpoolctl): n1 = n & -16 elements go through the vector
 * kernel (4 x 8-lane FMA accumulators over 32-blocks, folded to 4 x 4 lanes,
 * then 4 x 4-lane FMA over the remaining 16-blocks, lane-wise chain, then
 * (a0+a2)+(a1+a3)); the tail is a scalar FMA chain `dot += y[i] * x[i]`. */
static double ddot_skylakex(const double* x, const double* y, int64_t n) {
    int64_t n1 = n & -16, n32 = n1 & ~(int64_t)31, i = 0;
    double dot = 0.0;
    if (n1) {
        double acc[4][8], a4[4][4], a[4];
        memset(acc, 0, sizeof(acc));
        for (; i < n32; i += 32)
            for (int j = 0; j < 4; j++)
                for (int l = 0; l < 8; l++)
                    acc[j][l] = fma(x[i + 8 * j + l], y[i + 8 * j + l], acc[j][l]);
        for (int j = 0; j < 4; j++)
            for (int l = 0; l < 4; l++) a4[j][l] = acc[j][l] + acc[j][l + 4];
        for (; i < n1; i += 16)
            for (int j = 0; j < 4; j++)
                for (int l = 0; l < 4; l++)
                    a4[j][l] = fma(x[i + 4 * j + l], y[i + 4 * j + l], a4[j][l]);
        for (int l = 0; l < 4; l++) a[l] = ((a4[0][l] + a4[1][l]) + a4[2][l]) + a4[3][l];
        dot = (a[0] + a[2]) + (a[1] + a[3]);
    }
    for (; i < n; i++) dot = fma(y[i], x[i], dot);
    return dot;
}

/* The same library's Haswell core (also selected on Zen hosts), read from the
 * installed libscipy_openblas' ddot_kernel_8 / dot_compute for that core and
 * pinned against numpy under OPENBLAS_CORETYPE=Haswell (tests/golden/
 * make_golden.py haswell): 4 x 4-lane FMA accumulators over 16-blocks; each
 * folds its upper lane pair onto the lower, h_j = (acc_j[m] + acc_j[m+2]);
 * r = (h0 + h1) + (h2 + h3) per lane; dot = r0 + r1; the tail is an unfused
 * `dot += y[i] * x[i]` (product rounded, then the add). */
static double ddot_haswell(const double* x, const double* y, int64_t n) {
    int64_t n1 = n & -16, i = 0;
    double dot = 0.0;
    if (n1) {
        double acc[4][4];
        memset(acc, 0, sizeof(acc));
        for (; i < n1; i += 16)
            for (int j = 0; j < 4; j++)
                for (int l = 0; l < 4; l++)
                    acc[j][l] = fma(x[i + 4 * j + l], y[i + 4 * j + l], acc[j][l]);
        double r[2];
        for (int m = 0; m < 2; m++) {
            double h[4];
            for (int j = 0; j < 4; j++) h[j] = acc[j][m] + acc[j][m + 2];
            r[m] = (h[0] + h[1]) + (h[2] + h[3]);
        }
        dot = r[0] + r[1];
    }
    for (; i < n; i++) {
        double p = y[i] * x[i];
        dot = dot + p;
    }
    return dot;
}

static int g_dot_order = ORC_DOT_SKYLAKEX;

int orc_set_dot_order(int order) {
    if (order != ORC_DOT_SKYLAKEX && order != ORC_DOT_HASWELL) return -1;
    g_dot_order = order;
    return 0;
}

int orc_get_dot_order(void) { return g_dot_order; }

double orc_ddot(const double* x, const double* y, int64_t n) {
    return g_dot_order == ORC_DOT_HASWELL ? ddot_haswell(x, y, n) : ddot_skylakex(x, y, n);
}

/* workload.py:461-468 */
double orc_cosine(const double* a, const double* b, int64_t D) {
    double na = sqrt(orc_ddot(a, a, D));  /* np.linalg.norm = sqrt(x.dot(x)) */
    double nb = sqrt(orc_ddot(b, b, D));
    if (na == 0.0 && nb == 0.0) return 1.0;
    if (na == 0.0 || nb == 0.0) return 0.0;
    return orc_ddot(a, b, D) / (na * nb);
}

/* ---------------------------------------------------------------------------
 * Step 1: horizon selection
 * ------------------------------------------------------------------------- */

/* horizon.py:108-132, confidence branch (static branch is min(static_h, N)).
 * one_plus_t is the Python float `1.0 + cfg.threshold` (horizon.py:127). */
int32_t orc_decide_horizon_conf(const double* u, int64_t K, int64_t N,
                                double one_plus_t, int64_t min_horizon) {
    int64_t h_thresh = N;
    const double* fin = u + (K - 1) * N;
    for (int64_t n = 0; n < N; n++) {
        double m = orc_np_mean_col(u, K - 1, N, n);
        if (fin[n] > one_plus_t * m) { h_thresh = n; break; }  /* argmax of trips */
    }
    int64_t h = h_thresh > min_horizon ? h_thresh : min_horizon;
    return (int32_t)(h < N ? h : N);
}

/* workload.py:471-496 (validation lives in the Python wrapper). */
int64_t orc_round_optimal_horizon(const double* ref, int64_t Lr,
                                  const double* cand, int64_t Lc, int64_t D,
                                  double thr) {
    int64_t limit = Lr < Lc ? Lr : Lc;
    for (int64_t i = 0; i < limit; i++)
        if (orc_cosine(cand + i * D, ref + i * D, D) < thr) return i;
    return limit;
}

static void load_f64(double* dst, const void* src, int is_f64, int64_t off, int64_t cnt) {
    if (is_f64) {
        memcpy(dst, (const double*)src + off, (size_t)cnt * sizeof(double));
    } else {
        const float* s = (const float*)src + off;
        for (int64_t i = 0; i < cnt; i++) dst[i] = (double)s[i];
    }
}

static void set_threads(int nthreads) {
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
}

void orc_horizon_conf_batch(const void* U, int is_f64, int64_t R, int64_t K,
                            int64_t N, double one_plus_t, int64_t min_horizon,
                            int32_t* H, int nthreads) {
    set_threads(nthreads);
#pragma omp parallel
    {
        double* u = (double*)malloc((size_t)(K * N) * sizeof(double));
#pragma omp for schedule(static)
        for (int64_t r = 0; r < R; r++) {
            load_f64(u, U, is_f64, r * K * N, K * N);
            H[r] = orc_decide_horizon_conf(u, K, N, one_plus_t, min_horizon);
        }
        free(u);
    }
}

void orc_divergence_batch(const void* prev, const void* cand, int is_f64,
                          int64_t R, int64_t S, int64_t Lp, int64_t Lc,
                          int64_t D, const int32_t* offset,
                          const int32_t* len_prev, const int32_t* len_cand,
                          double thr, int32_t* H, double* cos, int nthreads) {
    set_threads(nthreads);
#pragma omp parallel
    {
        double* ref = (double*)malloc((size_t)(Lp * D + 1) * sizeof(double));
        double* cd = (double*)malloc((size_t)(Lc * D + 1) * sizeof(double));
#pragma omp for schedule(static)
        for (int64_t r = 0; r < R; r++) {
            int64_t off = offset ? offset[r] : 0;
            int64_t lp = len_prev ? len_prev[r] : Lp;
            int64_t lc = len_cand ? len_cand[r] : Lc;
            int64_t lr = lp - off;
            if (lr < 0) lr = 0;
            int64_t limit = lr < lc ? lr : lc;
            load_f64(ref, prev, is_f64, (r * Lp + off) * D, lr * D);
            int64_t best = limit;
            for (int64_t s = 0; s < S; s++) {
                load_f64(cd, cand, is_f64, ((r * S + s) * Lc) * D, lc * D);
                if (cos) {
                    double* c = cos + (r * S + s) * Lc;
                    for (int64_t i = 0; i < Lc; i++)
                        c[i] = i < limit ? orc_cosine(cd + i * D, ref + i * D, D) : NAN;
                }
                int64_t h = orc_round_optimal_horizon(ref, lr, cd, lc, D, thr);
                if (h < best) best = h;
            }
            H[r] = (int32_t)best;
        }
        free(ref);
        free(cd);
    }
}

/* ---------------------------------------------------------------------------
 * Step 2: execution-aware urgency
 * ------------------------------------------------------------------------- */

/* core.py:24-28 round_half_up + core.py:31-42 us_from_actions: the rational
 * count * 1e6 / (p/q) = X/Y with X = count*1e6*q, Y = p, rounded half-up as
 * (2X + Y) // (2Y) (invariant under the Fraction's gcd reduction). */
int64_t orc_us_from_actions(int64_t count, int64_t hz_num, int64_t hz_den) {
    __int128 X = (__int128)count * 1000000 * hz_den;
    __int128 Y = hz_num;
    return (int64_t)((2 * X + Y) / (2 * Y));
}

/* waiting.py:69-93: per round j < n_exec, gen-dominated (|G_j| >= |E_j|)
 * rounds take max(0, G_{j+1}.start - G_j.end) once G_{j+1} has started
 * (n_gen > j+1); exec-dominated rounds take max(0, E_{j+1}.start - E_j.end)
 * once E_{j+1} is recorded.  The final round accrues nothing. */
int64_t orc_total_wait(const int64_t* slots, int32_t n_exec, int32_t n_gen) {
    int64_t total = 0;
    for (int32_t j = 0; j < n_exec; j++) {
        const int64_t* s = slots + 4 * j;
        int64_t glen = s[1] - s[0], elen = s[3] - s[2];
        if (glen >= elen) {
            if (n_gen > j + 1) {
                int64_t w = slots[4 * (j + 1) + 0] - s[1];
                total += w > 0 ? w : 0;
            }
        } else if (j + 1 < n_exec) {
            int64_t w = slots[4 * (j + 1) + 2] - s[3];
            total += w > 0 ? w : 0;
        }
    }
    return total;
}

/* waiting.py:96-100 and waiting.py:62-66.  Python int / int is the correctly
 * rounded quotient, equal to the fp64 division for operands below 2^53. */
double orc_current_wait_ratio(int64_t total_wait, int64_t t_start, int64_t now) {
    if (now <= t_start) return 0.0;
    double r = (double)total_wait / (double)(now - t_start);
    r = r > 0.0 ? r : 0.0;
    return r < 1.0 ? r : 1.0;
}

/* scheduler.py:79-88 */
int32_t orc_assign_bucket(double wr, int64_t skipped, int64_t buckets,
                          int64_t aging_interval) {
    int64_t b = (int64_t)floor(wr * (double)buckets);
    if (b > buckets - 1) b = buckets - 1;
    if (skipped >= aging_interval) {
        b = b + skipped / aging_interval;
        if (b > buckets - 1) b = buckets - 1;
    }
    return (int32_t)b;
}

/* ---------------------------------------------------------------------------
 * Step 3: ordering and edge admission (scheduler.py:107-157, 193-276)
 * ------------------------------------------------------------------------- */

typedef struct {
    int64_t k0, k1, k2;  /* composite sort key */
    int32_t rank;        /* task_id order */
    int32_t idx;
} orc_item;

static int cmp_item(const void* pa, const void* pb) {
    const orc_item* a = (const orc_item*)pa;
    const orc_item* b = (const orc_item*)pb;
    if (a->k0 != b->k0) return a->k0 < b->k0 ? -1 : 1;
    if (a->k1 != b->k1) return a->k1 < b->k1 ? -1 : 1;
    if (a->k2 != b->k2) return a->k2 < b->k2 ? -1 : 1;
    if (a->rank != b->rank) return a->rank < b->rank ? -1 : 1;
    return 0;
}

int64_t orc_plan(const orc_fleet* f, int policy, int64_t buckets,
                 int64_t aging_interval, int64_t stale_threshold,
                 int64_t default_exec_estimate, int64_t now, int64_t hz_num,
                 int64_t hz_den, int64_t edge_avail, int32_t* order,
                 int64_t* total_wait, double* wr_out, int32_t* bucket_out,
                 int64_t* est_out, int64_t* need_time, uint8_t* admitted,
                 uint8_t* refetch, int32_t* skipped_out) {
    int64_t n = f->n;
    orc_item* items = (orc_item*)malloc((size_t)(n > 0 ? n : 1) * sizeof(orc_item));
    int64_t* bkt = (int64_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
    for (int64_t i = 0; i < n; i++) {
        const int64_t* sl = f->slots + 4 * f->hist_off[i];
        /* scheduler.py:91-104 estimate_exec_latency: last exec length */
        int64_t est = f->n_exec[i] > 0
                          ? sl[4 * (f->n_exec[i] - 1) + 3] - sl[4 * (f->n_exec[i] - 1) + 2]
                          : default_exec_estimate;
        int64_t w = orc_total_wait(sl, f->n_exec[i], f->n_gen[i]);
        double wr = orc_current_wait_ratio(w, f->t_start[i], now);
        int32_t b = orc_assign_bucket(wr, f->skipped[i], buckets, aging_interval);
        if (total_wait) total_wait[i] = w;
        if (wr_out) wr_out[i] = wr;
        if (bucket_out) bucket_out[i] = b;
        if (est_out) est_out[i] = est;
        /* core.py:157-166 exec_end_from_piggyback: the next-need instant */
        if (need_time)
            need_time[i] = f->issued_at[i] + orc_us_from_actions(f->remaining[i], hz_num, hz_den);
        items[i].rank = f->lexrank[i];
        items[i].idx = (int32_t)i;
        bkt[i] = b;
        if (policy == ORC_KAIROS) {
            /* scheduler.py:113-115 key (-aged, issued_at, task_id) */
            items[i].k0 = -(est * (1 + (int64_t)f->skipped[i]));
            items[i].k1 = f->issued_at[i];
            items[i].k2 = 0;
        } else if (policy == ORC_FIFO) {
            /* scheduler.py:143-144 */
            items[i].k0 = f->issued_at[i];
            items[i].k1 = 0;
            items[i].k2 = 0;
        } else {
            /* scheduler.py:147-157 */
            items[i].k0 = f->accum_gen[i];
            items[i].k1 = f->issued_at[i];
            items[i].k2 = 0;
        }
    }
    int64_t pos = 0;
    if (policy == ORC_KAIROS) {
        /* scheduler.py:130-140: buckets high -> low, each sorted */
        orc_item* tmp = (orc_item*)malloc((size_t)(n > 0 ? n : 1) * sizeof(orc_item));
        for (int64_t b = buckets - 1; b >= 0; b--) {
            int64_t m = 0;
            for (int64_t i = 0; i < n; i++)
                if (bkt[i] == b) tmp[m++] = items[i];
            qsort(tmp, (size_t)m, sizeof(orc_item), cmp_item);
            for (int64_t i = 0; i < m; i++) order[pos++] = tmp[i].idx;
        }
        free(tmp);
    } else {
        qsort(items, (size_t)n, sizeof(orc_item), cmp_item);
        for (int64_t i = 0; i < n; i++) order[pos++] = items[i].idx;
    }
    /* scheduler.py:204-207 edge prefix; 223-234 refetch + skip counters */
    int64_t n_edge = edge_avail < 0 ? 0 : (edge_avail < n ? edge_avail : n);
    for (int64_t p = 0; p < n; p++) {
        int32_t i = order[p];
        int in = p < n_edge;
        if (admitted) admitted[i] = (uint8_t)in;
        if (refetch) refetch[i] = (uint8_t)(in && (now - f->obs_captured_at[i] > stale_threshold));
        if (skipped_out) skipped_out[i] = in ? 0 : f->skipped[i] + 1;
    }
    free(items);
    free(bkt);
    return n_edge;
}

/* ---------------------------------------------------------------------------
 * Phase 3: hybrid placement (scheduler.py:160-241, engines.py:132-169)
 * ------------------------------------------------------------------------- */

/* engines.py:132-155: exact at profiled points, linear interpolation between
 * them rounded half-up (lat_lo is an integer, so only the fraction rounds). */
int64_t orc_batch_latency(const orc_profile* p, int64_t batch) {
    if (batch <= p->batch[0]) return p->latency[0];
    for (int32_t i = 0; i + 1 < p->npts; i++) {
        int64_t blo = p->batch[i], bhi = p->batch[i + 1];
        int64_t llo = p->latency[i], lhi = p->latency[i + 1];
        if (batch == bhi) return lhi;
        if (blo < batch && batch < bhi) {
            __int128 num = (__int128)(lhi - llo) * (batch - blo), den = bhi - blo;
            return llo + (int64_t)((2 * num + den) / (2 * den));
        }
    }
    return p->latency[p->npts - 1];
}

/* engines.py:158-169: base latency + round_half_up(bytes * 8e6 / bps). */
int64_t orc_transfer_time(const orc_net* net, int64_t payload_bytes, int up) {
    int64_t bps = up ? net->uplink_bps : net->downlink_bps;
    __int128 num = (__int128)payload_bytes * 8 * 1000000;
    return net->base_latency_us + (int64_t)((2 * num + bps) / (2 * (__int128)bps));
}

/* scheduler.py:160-164 */
static int64_t orc_drain(const orc_profile* p, int64_t queued) {
    if (queued <= 0) return 0;
    int64_t waves = (queued + p->max_batch - 1) / p->max_batch;
    return waves * orc_batch_latency(p, p->max_batch);
}

int64_t orc_plan_tiers(const orc_fleet* f, const int64_t* payload, int policy, int64_t buckets,
                       int64_t aging_interval, int64_t stale_threshold,
                       int64_t default_exec_estimate, int64_t now, const orc_profile* edge,
                       const orc_profile* cloud, const orc_net* net, int64_t edge_in_flight,
                       int64_t cloud_in_flight, int32_t* order, uint8_t* tier,
                       int32_t* cloud_order, uint8_t* refetch, int32_t* skipped_out,
                       int64_t* n_edge_out) {
    int64_t n = f->n;
    /* phases 1-2: the reference order (orc_plan with no edge budget) */
    orc_plan(f, policy, buckets, aging_interval, stale_threshold, default_exec_estimate, now, 30,
             1, 0, order, NULL, NULL, NULL, NULL, NULL, NULL, NULL, NULL);
    /* scheduler.py:204-207 */
    int64_t edge_avail = edge ? edge->capacity - edge_in_flight : 0;
    int64_t cloud_avail = cloud ? cloud->capacity - cloud_in_flight : 0;
    if (edge_avail < 0) edge_avail = 0;
    if (cloud_avail < 0) cloud_avail = 0;
    int64_t n_edge = edge_avail < n ? edge_avail : n;
    for (int64_t p = 0; p < n; p++) tier[order[p]] = p < n_edge ? 1 : 0;
    /* scheduler.py:210-221: greedy cloud offload over the rest, in order */
    int64_t n_cloud = 0;
    int64_t planned_edge = n_edge;
    for (int64_t p = n_edge; p < n; p++) {
        int32_t i = order[p];
        if (!cloud || !net || n_cloud >= cloud_avail) continue;
        int has_edge = edge != NULL;
        int64_t edge_est = 0;
        if (has_edge) {  /* _edge_estimate (scheduler.py:167-174) */
            int64_t own = planned_edge > 1 ? planned_edge : 1;
            if (own > edge->max_batch) own = edge->max_batch;
            edge_est = orc_drain(edge, edge_in_flight + planned_edge) + orc_batch_latency(edge, own);
        }
        /* _cloud_estimate (scheduler.py:177-190) */
        int64_t own_c = n_cloud + 1 < cloud->max_batch ? n_cloud + 1 : cloud->max_batch;
        int64_t cloud_est = orc_drain(cloud, cloud_in_flight + n_cloud) +
                            orc_transfer_time(net, payload[i], 1) + orc_batch_latency(cloud, own_c) +
                            orc_transfer_time(net, 0, 0);
        if (!has_edge || cloud_est < edge_est) {
            tier[i] = 2;
            cloud_order[n_cloud++] = i;
        }
    }
    /* scheduler.py:223-234 */
    for (int64_t i = 0; i < n; i++) {
        int disp = tier[i] != 0;
        refetch[i] = (uint8_t)(disp && (now - f->obs_captured_at[i] > stale_threshold));
        skipped_out[i] = disp ? 0 : f->skipped[i] + 1;
    }
    *n_edge_out = n_edge;
    return n_cloud;
}
