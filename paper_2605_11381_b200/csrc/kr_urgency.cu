// kr_urgency.cu -- step 2 of the decision core: execution-aware urgency.
//
// One fused elementwise pass per pending request (thread per request):
//   ledger_from_history   waiting.py:69-93  (CSR history slots, in-flight successor)
//   current_wait_ratio    waiting.py:96-100, 62-66
//   assign_bucket         scheduler.py:79-88 (wait-ratio bucket + skip aging)
//   estimate_exec_latency scheduler.py:91-104 (last execution length = projected
//                         execution duration of the next round)
//   aged estimate + order scheduler.py:113-115, 130-140 (packed 128-bit key)
//   next-need time        core.py:157-166 exec_end_from_piggyback: issue time plus
//                         the remaining actions at the control rate
// Integer-µs everywhere except the wait ratio (one fp64 division, correctly
// rounded like Python's int / int) and its bucket multiply.
#include "kr_common.cuh"
#include "kr_host.cuh"
#include "kr_select_state.cuh"

namespace kr {

__global__ void k_us_from_actions(const int64_t* count, const int64_t* base, int64_t n,
                                  int64_t hz_num, int64_t hz_den, int64_t* out, uint32_t* flags) {
    uint32_t fl = 0;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        int64_t us = us_from_actions(count[i], hz_num, hz_den, &fl);
        out[i] = (base ? base[i] : 0) + us;
    }
    if (fl && flags) atomicOr(flags, fl);
}

__global__ void k_wait_ratio(const int64_t* total, const int64_t* t_start, int64_t n, int64_t now,
                             double* wr, uint32_t* flags) {
    uint32_t fl = 0;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x)
        wr[i] = wait_ratio(total[i], t_start[i], now, &fl);
    if (fl && flags) atomicOr(flags, fl);
}

__global__ void k_assign_bucket(const double* wr, const int32_t* skipped, int64_t n, int32_t B,
                                int32_t A, int32_t* bucket) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x)
        bucket[i] = assign_bucket(wr[i], skipped[i], B, A);
}

struct UrgencyOut {
    kr_key* keys;
    int64_t* need_time;
    int64_t* total_wait;
    double* wr;
    int32_t* bucket;
    int64_t* est;
    int64_t* slot_wait;
    unsigned long long* key_stats;
    uint32_t* flags;
    SelState* sel = nullptr;  // kr_urgency_prep: the last CTA prepares the select state
    int64_t sel_k = 0;
    unsigned long long* sel_part = nullptr;  // [gridDim][4] per-CTA key statistics (prep)
};

// Per-round waits of one request (WaitLedger.waits), -1 where none recorded.
__device__ __forceinline__ void slot_waits(const int64_t* slots, int32_t n_exec, int32_t n_gen,
                                           int64_t* out) {
    for (int32_t j = 0; j < n_exec; j++) {
        Slot cur = load_slot(slots, j);
        int64_t w = -1;
        if (cur.ge - cur.gs >= cur.ee - cur.es) {
            if (n_gen > j + 1) {
                w = load_slot(slots, j + 1).gs - cur.ge;
                w = w > 0 ? w : 0;
            }
        } else if (j + 1 < n_exec) {
            w = load_slot(slots, j + 1).es - cur.ee;
            w = w > 0 ? w : 0;
        }
        out[j] = w;
    }
}


// Per-request inputs of the urgency pass.  FleetSrc: one self-contained
// structure-of-arrays per planning round (history as CSR slots, walked per
// request).  LedgerSrc: the device-resident incremental ledger -- requests
// index their task, whose running wait total and last execution are O(1).
struct FleetSrc {
    kr_fleet f;
    static constexpr bool kSlots = true;
    __device__ int64_t n() const { return f.n; }
    __device__ int64_t issued(int64_t i) const { return __ldg(f.issued_at + i); }
    __device__ int32_t rank(int64_t i) const { return __ldg(f.lexrank + i); }
    __device__ int32_t remaining(int64_t i) const { return __ldg(f.remaining + i); }
    __device__ int64_t accum(int64_t i) const { return __ldg(f.accum_gen + i); }
    __device__ int32_t skipped(int64_t i) const { return f.skipped[i]; }
    // total wait, t_start, number of executions and the last execution length
    __device__ void hist(int64_t i, int64_t& w, int64_t& t0, int32_t& ne, int64_t& last) const {
        const int64_t* slots = f.slots + 4 * __ldg(f.hist_off + i);
        ne = __ldg(f.n_exec + i);
        t0 = __ldg(f.t_start + i);
        history_walk(slots, ne, __ldg(f.n_gen + i), w, last);
    }
    __device__ void waits(int64_t i, int64_t* out) const {
        slot_waits(f.slots + 4 * __ldg(f.hist_off + i), __ldg(f.n_exec + i), __ldg(f.n_gen + i),
                   out + __ldg(f.hist_off + i));
    }
    // L2 prefetch of request i's fields (its history span follows in slots_l2)
    __device__ __forceinline__ int64_t fields_l2(int64_t i) const {
        l2_prefetch(f.issued_at + i);
        l2_prefetch(f.lexrank + i);
        l2_prefetch(f.remaining + i);
        l2_prefetch(f.skipped + i);
        l2_prefetch(f.n_exec + i);
        l2_prefetch(f.n_gen + i);
        l2_prefetch(f.t_start + i);
        return __ldg(f.hist_off + i);
    }
    __device__ __forceinline__ void slots_l2(int64_t off) const {
        const int64_t* p = f.slots + 4 * off;
        l2_prefetch(p);
        l2_prefetch(p + 16);  // the next 128 bytes (histories of more than 4 slots are rare)
    }
};

struct LedgerSrc {
    kr_ledger L;
    kr_requests q;
    static constexpr bool kSlots = false;
    __device__ int64_t n() const { return q.n; }
    __device__ int64_t issued(int64_t i) const { return __ldg(q.issued_at + i); }
    __device__ int32_t rank(int64_t i) const { return __ldg(q.lexrank + i); }
    __device__ int32_t remaining(int64_t i) const { return __ldg(q.remaining + i); }
    __device__ int64_t accum(int64_t i) const { return __ldg(q.accum_gen + i); }
    __device__ int32_t skipped(int64_t i) const { return q.skipped[i]; }
    __device__ void hist(int64_t i, int64_t& w, int64_t& t0, int32_t& ne, int64_t& last) const {
        const int64_t t = __ldg(q.task + i);
        ne = L.n_exec[t];
        w = L.wait_total[t];
        t0 = L.t_start[t];
        if (ne > 0) {
            const int64_t* sl = L.slots + (t * L.cap + ne - 1) * 4;
            last = sl[3] - sl[2];
        }
    }
    __device__ void waits(int64_t, int64_t*) const {}
    __device__ __forceinline__ int64_t fields_l2(int64_t) const { return 0; }
    __device__ __forceinline__ void slots_l2(int64_t) const {}
};

// Per-launch constants of the urgency pass, prepared on the host from kr_sched:
// the aging interval as a multiply-shift divisor and, for an integer control
// rate, the reciprocal of the round-half-up denominator 2*hz.
struct UrgConst {
    FastDiv aging;
    double rinv;    // 1 / (2 hz)      (fast_time only)
    int64_t den;    // 2 hz            (fast_time only)
    int fast_time;  // hz_den == 1 && hz_num < 2^40
};
static UrgConst urg_const(const kr_sched& c) {
    UrgConst u{};
    u.aging = make_fastdiv(static_cast<uint32_t>(c.aging_interval));
    u.fast_time = c.hz_den == 1 && c.hz_num < (int64_t(1) << 40);
    u.den = 2 * c.hz_num;
    u.rinv = 1.0 / static_cast<double>(u.den);
    return u;
}

// us_from_actions for an int32 action count: the integer-hz branch's
// (2*count*10^6 + hz) / (2 hz) via the fp64 reciprocal and one exact integer
// correction (the numerator is below 2^53, the estimate within one of the
// quotient); otherwise the general __int128 path.
__device__ __forceinline__ int64_t us_from_actions32(int32_t count, const kr_sched& c,
                                                     const UrgConst& u, uint32_t* flag_bits) {
    if (!u.fast_time || count < 0) return us_from_actions(count, c.hz_num, c.hz_den, flag_bits);
    const int64_t num = static_cast<int64_t>(count) * 2000000 + c.hz_num;
    int64_t q = static_cast<int64_t>(__dmul_rn(static_cast<double>(num), u.rinv));
    const int64_t r = num - q * u.den;
    q += r < 0 ? -1 : (r >= u.den ? 1 : 0);
    return q;
}

// assign_bucket (scheduler.py:79-88) with the aging division by multiply-shift
// (skipped >= A >= 1 here, so the dividend is a non-negative int32).
__device__ __forceinline__ int32_t assign_bucket32(double wr, int32_t skipped, int32_t B, int32_t A,
                                                   const FastDiv& fa) {
    int32_t b = static_cast<int32_t>(floor(dmul(wr, static_cast<double>(B))));
    if (b > B - 1) b = B - 1;
    if (skipped >= A) {
        b = b + static_cast<int32_t>(fdiv(static_cast<uint32_t>(skipped), fa));
        if (b > B - 1) b = B - 1;
    }
    return b;
}

// One request: its packed key (and the optional intermediates / need time).
// LEAN: the planning round's case decided at compile time -- Kairos keys, the
// need time, no intermediates -- so no per-request policy or output tests.
template <class Src, bool LEAN = false>
__device__ __forceinline__ kr_key urgency_one(const Src& s, const kr_sched& c, const UrgConst& u,
                                              const UrgencyOut& o, int64_t i, uint32_t& fl) {
    const int64_t issued = s.issued(i);
    const int32_t rank = s.rank(i);
    const int32_t policy = LEAN ? KR_KAIROS : c.policy;
    if (LEAN || o.need_time) {
        int32_t rem = s.remaining(i);
        o.need_time[i] = issued + us_from_actions32(rem, c, u, &fl);
    }
    kr_key key;
    if (policy == KR_FIFO) {
        key.hi = static_cast<uint64_t>(issued) ^ (uint64_t(1) << 63);
        key.lo = static_cast<uint64_t>(static_cast<uint32_t>(rank));
        if (rank < 0) fl |= KR_FLAG_KEY_RANGE;
    } else if (policy == KR_LAS) {
        key.hi = static_cast<uint64_t>(s.accum(i)) ^ (uint64_t(1) << 63);
        key.lo = issued_rank_word(issued, c.issued_base, rank, &fl);
    }
    const bool need_hist =
        policy == KR_KAIROS || (!LEAN && (o.total_wait || o.wr || o.bucket || o.est || o.slot_wait));
    if (need_hist) {
        const int32_t skipped = s.skipped(i);
        int64_t w, t0, last = 0;
        int32_t ne;
        s.hist(i, w, t0, ne, last);
        double wr = wait_ratio(w, t0, c.now, &fl);
        int32_t b = assign_bucket32(wr, skipped, c.buckets, c.aging_interval, u.aging);
        const int64_t est = ne > 0 ? last : c.default_exec_estimate;
        if constexpr (!LEAN) {
            if (o.total_wait) o.total_wait[i] = w;
            if (o.wr) o.wr[i] = wr;
            if (o.bucket) o.bucket[i] = b;
            if (o.est) o.est[i] = est;
            if constexpr (Src::kSlots)
                if (o.slot_wait) s.waits(i, o.slot_wait);
        }
        if (policy == KR_KAIROS) {
            // aged = est * (1 + skipped), descending -> stored complemented;
            // clamped at 2^56 - 1 (the 128-bit product of the original
            // formulation: a negative multiplier wraps to a huge value)
            const uint64_t e = est < 0 ? 0 : static_cast<uint64_t>(est);
            const int64_t m = 1 + static_cast<int64_t>(skipped);
            bool over;
            uint64_t a;
            if (m >= 0) {
                const uint64_t lo = e * static_cast<uint64_t>(m);
                over = __umul64hi(e, static_cast<uint64_t>(m)) != 0 || lo > kAgedMask;
                a = over ? kAgedMask : lo;
            } else {
                over = e != 0;
                a = over ? kAgedMask : 0;
            }
            if (est < 0 || skipped < 0 || over) fl |= KR_FLAG_KEY_RANGE;
            key.hi = (static_cast<uint64_t>(c.buckets - 1 - b) << 56) | (kAgedMask - a);
            key.lo = issued_rank_word(issued, c.issued_base, rank, &fl);
        }
    }
    return key;
}

#ifndef KR_URG_MINB
#define KR_URG_MINB 4  // resident CTAs per SM the register budget is sized for
#endif
template <class Src, class Idx, bool LEAN = false>
__global__ void __launch_bounds__(256, KR_URG_MINB) k_urgency(Src s, kr_sched c, UrgConst u,
                                                              UrgencyOut o) {
    griddep_wait();  // programmatic dependent launch (kr_host.cuh launch_pdl)
    // select statistics (OR / AND of the keys) per thread, then per warp and
    // block (a per-iteration redux.sync variant measured 4% slower)
    __shared__ uint32_t red[8];  // OR hi.hi, hi.lo, lo.hi, lo.lo | AND (same order)
    if (threadIdx.x < 8) red[threadIdx.x] = threadIdx.x < 4 ? 0u : ~0u;
    __syncthreads();
    uint32_t fl = 0;
    const Idx n = static_cast<Idx>(s.n());
    const bool stats = o.key_stats != nullptr;
    unsigned long long ohi = 0, olo = 0, ahi = ~0ull, alo = ~0ull;
    const Idx stride = Idx(gridDim.x) * blockDim.x;
    for (Idx i = blockIdx.x * Idx(blockDim.x) + threadIdx.x; i < n; i += stride) {
        // the next request's fields into L2 now, its history span after this
        // request is done: the next iteration's two dependent loads hit L2
        const Idx nx = i + stride;
        int64_t off_nx = 0;
        if (Src::kSlots && nx < n) off_nx = s.fields_l2(nx);
        const kr_key key = urgency_one<Src, LEAN>(s, c, u, o, i, fl);
        if (Src::kSlots && nx < n) s.slots_l2(off_nx);
        o.keys[i] = key;
        ohi |= key.hi; olo |= key.lo; ahi &= key.hi; alo &= key.lo;
    }
    if (stats) {  // warp-reduced, then eight shared words per block
#pragma unroll
        for (int t = 16; t; t >>= 1) {
            ohi |= __shfl_xor_sync(0xffffffffu, ohi, t); olo |= __shfl_xor_sync(0xffffffffu, olo, t);
            ahi &= __shfl_xor_sync(0xffffffffu, ahi, t); alo &= __shfl_xor_sync(0xffffffffu, alo, t);
        }
        if ((threadIdx.x & 31) == 0) {
            atomicOr(&red[0], static_cast<uint32_t>(ohi >> 32)); atomicOr(&red[1], static_cast<uint32_t>(ohi));
            atomicOr(&red[2], static_cast<uint32_t>(olo >> 32)); atomicOr(&red[3], static_cast<uint32_t>(olo));
            atomicAnd(&red[4], static_cast<uint32_t>(ahi >> 32)); atomicAnd(&red[5], static_cast<uint32_t>(ahi));
            atomicAnd(&red[6], static_cast<uint32_t>(alo >> 32)); atomicAnd(&red[7], static_cast<uint32_t>(alo));
        }
    }
    if (fl && o.flags) atomicOr(o.flags, fl);
    if (o.sel) {
        // prep: each CTA stores its partial statistics (no contended atomics);
        // the last CTA to finish reduces them into the select state
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long* pp = o.sel_part + 4 * blockIdx.x;
            pp[0] = (static_cast<unsigned long long>(red[0]) << 32) | red[1];
            pp[1] = (static_cast<unsigned long long>(red[2]) << 32) | red[3];
            pp[2] = (static_cast<unsigned long long>(red[4]) << 32) | red[5];
            pp[3] = (static_cast<unsigned long long>(red[6]) << 32) | red[7];
        }
        __shared__ bool last;
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) last = atomicAdd(&o.sel->done_urg, 1u) == gridDim.x - 1;
        __syncthreads();
        if (last) {
            __threadfence();
            unsigned long long a = 0, b = 0, c = ~0ull, d = ~0ull;
            for (unsigned g = threadIdx.x; g < gridDim.x; g += blockDim.x) {
                const ulonglong2 v0 = __ldcg(reinterpret_cast<const ulonglong2*>(o.sel_part + 4 * g));
                const ulonglong2 v1 = __ldcg(reinterpret_cast<const ulonglong2*>(o.sel_part + 4 * g + 2));
                a |= v0.x; b |= v0.y; c &= v1.x; d &= v1.y;
            }
#pragma unroll
            for (int t = 16; t; t >>= 1) {
                a |= __shfl_xor_sync(0xffffffffu, a, t); b |= __shfl_xor_sync(0xffffffffu, b, t);
                c &= __shfl_xor_sync(0xffffffffu, c, t); d &= __shfl_xor_sync(0xffffffffu, d, t);
            }
            __shared__ unsigned long long wred[4][8];
            const int wp = threadIdx.x >> 5;
            if ((threadIdx.x & 31) == 0) { wred[0][wp] = a; wred[1][wp] = b; wred[2][wp] = c; wred[3][wp] = d; }
            __syncthreads();
            if (threadIdx.x == 0) {
                for (int w = 1; w < static_cast<int>(blockDim.x >> 5); w++) {
                    a |= wred[0][w]; b |= wred[1][w]; c &= wred[2][w]; d &= wred[3][w];
                }
                wred[0][0] = a; wred[1][0] = b; wred[2][0] = c; wred[3][0] = d;
            }
            __syncthreads();
            const unsigned long long st4[4] = {wred[0][0], wred[1][0], wred[2][0], wred[3][0]};
            sel_prepare(o.sel, s.n(), o.sel_k, st4, o.keys);
        }
        return;
    }
    if (stats) {
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned long long ohi = (static_cast<unsigned long long>(red[0]) << 32) | red[1];
            const unsigned long long olo = (static_cast<unsigned long long>(red[2]) << 32) | red[3];
            const unsigned long long ahi = (static_cast<unsigned long long>(red[4]) << 32) | red[5];
            const unsigned long long alo = (static_cast<unsigned long long>(red[6]) << 32) | red[7];
            if (ohi) atomicOr(&o.key_stats[0], ohi);
            if (olo) atomicOr(&o.key_stats[1], olo);
            if (~ahi) atomicAnd(&o.key_stats[2], ahi);
            if (~alo) atomicAnd(&o.key_stats[3], alo);
        }
    }
}

static unsigned grid_for(int64_t n, int threads) {
    int64_t b = (n + threads - 1) / threads;
    int64_t cap = static_cast<int64_t>(device_info().sm_count) * 8;
    if (b > cap) b = cap;
    return static_cast<unsigned>(b < 1 ? 1 : b);
}

// Persistent grid: every CTA resident at once (SMs x occupancy), each thread
// looping over several requests so the block-level key statistics amortise;
// 32-bit indices below 2^31 requests.
template <class Src>
static void launch_urgency(const Src& src, int64_t n, const kr_sched& c, const UrgencyOut& o,
                           cudaStream_t st) {
    const UrgConst u = urg_const(c);
    static const bool lean_off = std::getenv("KR_URG_NO_LEAN") != nullptr;  // A/B knob
    const bool lean = !lean_off && c.policy == KR_KAIROS && o.need_time && !o.total_wait && !o.wr &&
                      !o.bucket && !o.est && !o.slot_wait;
    if (lean && n < (int64_t(1) << 31)) {
        static int per_sm = occupancy(k_urgency<Src, int32_t, true>, 256);
        launch_pdl(k_urgency<Src, int32_t, true>, grid_cap(n, 256, per_sm), 256, st, src, c, u, o);
    } else if (n < (int64_t(1) << 31)) {
        static int per_sm = occupancy(k_urgency<Src, int32_t>, 256);
        launch_pdl(k_urgency<Src, int32_t, false>, grid_cap(n, 256, per_sm), 256, st, src, c, u, o);
    } else {
        static int per_sm = occupancy(k_urgency<Src, int64_t>, 256);
        launch_pdl(k_urgency<Src, int64_t, false>, grid_cap(n, 256, per_sm), 256, st, src, c, u, o);
    }
}

}  // namespace kr

using namespace kr;

extern "C" int kr_us_from_actions(const int64_t* count, const int64_t* base, int64_t n,
                                  int64_t hz_num, int64_t hz_den, int64_t* out, uint32_t* flags,
                                  void* stream) {
    if (n < 0 || hz_num <= 0 || hz_den <= 0) return KR_EINVAL;
    if (n == 0) return KR_OK;
    if (!count || !out) return KR_EINVAL;
    k_us_from_actions<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(count, base, n, hz_num,
                                                                        hz_den, out, flags);
    return check_launch("kr_us_from_actions");
}

extern "C" int kr_wait_ratio(const int64_t* total_wait, const int64_t* t_start, int64_t n,
                             int64_t now, double* wr, uint32_t* flags, void* stream) {
    if (n < 0) return KR_EINVAL;
    if (n == 0) return KR_OK;
    if (!total_wait || !t_start || !wr) return KR_EINVAL;
    k_wait_ratio<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(total_wait, t_start, n, now, wr,
                                                                   flags);
    return check_launch("kr_wait_ratio");
}

extern "C" int kr_assign_bucket(const double* wr, const int32_t* skipped, int64_t n,
                                int32_t buckets, int32_t aging_interval, int32_t* bucket,
                                void* stream) {
    if (n < 0 || buckets < 1 || aging_interval < 1) return KR_EINVAL;
    if (n == 0) return KR_OK;
    if (!wr || !skipped || !bucket) return KR_EINVAL;
    k_assign_bucket<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(wr, skipped, n, buckets,
                                                                      aging_interval, bucket);
    return check_launch("kr_assign_bucket");
}

extern "C" int kr_urgency(const kr_fleet* fleet, const kr_sched* cfg, kr_key* keys,
                          int64_t* need_time, int64_t* total_wait, double* wr, int32_t* bucket,
                          int64_t* est, int64_t* slot_wait, unsigned long long* key_stats,
                          uint32_t* flags, void* stream) {
    if (!fleet || !cfg || fleet->n < 0) return KR_EINVAL;
    if (cfg->policy < KR_KAIROS || cfg->policy > KR_LAS || cfg->buckets < 1 ||
        cfg->buckets > 256 || cfg->aging_interval < 1 || cfg->hz_num <= 0 || cfg->hz_den <= 0)
        return KR_EINVAL;
    if (fleet->n == 0) return KR_OK;
    if (!keys) return KR_EINVAL;
    UrgencyOut o{keys, need_time, total_wait, wr, bucket, est, slot_wait, key_stats, flags};
    launch_urgency(FleetSrc{*fleet}, fleet->n, *cfg, o, as_stream(stream));
    return check_launch("kr_urgency");
}

extern "C" int kr_urgency_prep(const kr_fleet* fleet, const kr_sched* cfg, kr_key* keys,
                               int64_t* need_time, uint32_t* flags, int64_t k, void* ws,
                               size_t ws_bytes, void* stream) {
    if (!fleet || !cfg || fleet->n < (int64_t(1) << 14) || k < 0) return KR_EINVAL;
    if (cfg->policy < KR_KAIROS || cfg->policy > KR_LAS || cfg->buckets < 1 ||
        cfg->buckets > 256 || cfg->aging_interval < 1 || cfg->hz_num <= 0 || cfg->hz_den <= 0)
        return KR_EINVAL;
    if (!keys || !ws || ws_bytes < sizeof(SelState)) return KR_EINVAL;
    // kr_select.cu carve(): the state heads the workspace, the level-0 digit
    // array (n x 2 bytes, written only by the select) follows 256-byte aligned;
    // it holds the per-CTA statistics meanwhile (grid x 32 bytes <= n x 2)
    unsigned char* base = static_cast<unsigned char*>(ws);
    const size_t off = (sizeof(SelState) + 255) & ~size_t(255);
    UrgencyOut o{keys, need_time, nullptr, nullptr, nullptr, nullptr, nullptr,
                 reinterpret_cast<unsigned long long*>(base + off), flags};
    o.sel = reinterpret_cast<SelState*>(base);
    o.sel_k = k;
    o.sel_part = reinterpret_cast<unsigned long long*>(base + off);
    launch_urgency(FleetSrc{*fleet}, fleet->n, *cfg, o, as_stream(stream));
    return check_launch("kr_urgency_prep");
}

extern "C" int kr_urgency_ledger(const kr_ledger* ledger, const kr_requests* req,
                                 const kr_sched* cfg, kr_key* keys, int64_t* need_time,
                                 int64_t* total_wait, double* wr, int32_t* bucket, int64_t* est,
                                 unsigned long long* key_stats, uint32_t* flags, void* stream) {
    if (!ledger || !req || !cfg || req->n < 0 || ledger->cap < 1) return KR_EINVAL;
    if (cfg->policy < KR_KAIROS || cfg->policy > KR_LAS || cfg->buckets < 1 ||
        cfg->buckets > 256 || cfg->aging_interval < 1 || cfg->hz_num <= 0 || cfg->hz_den <= 0)
        return KR_EINVAL;
    if (req->n == 0) return KR_OK;
    if (!keys || !req->task) return KR_EINVAL;
    UrgencyOut o{keys, need_time, total_wait, wr, bucket, est, nullptr, key_stats, flags};
    launch_urgency(LedgerSrc{*ledger, *req}, req->n, *cfg, o, as_stream(stream));
    return check_launch("kr_urgency_ledger");
}

// ---------------------------------------------------------------------------
// Incremental ledger (core.py:169-249 TaskState mutations, waiting.py:69-93)
// ---------------------------------------------------------------------------
// One thread per touched task applies that task's events in order.  A round
// j's wait becomes final the moment it is first computable (its successor's
// generation start on the gen-dominated branch, its successor's execution on
// the exec-dominated one), and the computable rounds always form a prefix, so
// wait_total advances a cursor (wait_next) instead of re-walking the history.
namespace kr {
__global__ void k_ledger_apply(kr_ledger L, kr_events ev, uint32_t* flags) {
    uint32_t fl = 0;
    for (int64_t g = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; g < ev.n_groups;
         g += int64_t(gridDim.x) * blockDim.x) {
        const int64_t t = ev.task[g];
        if (t < 0 || t >= L.n_tasks) {
            fl |= KR_FLAG_LEDGER;
            continue;
        }
        int64_t* sl = L.slots + t * L.cap * 4;
        int32_t ne = L.n_exec[t], ng = L.n_gen[t], jw = L.wait_next[t];
        int64_t w = L.wait_total[t];
        for (int32_t e = ev.off[g]; e < ev.off[g + 1]; e++) {
            const int32_t k = ev.kind[e], j = ev.round[e];
            const int64_t a = ev.a[e];
            if (k == KR_EV_NEW) {
                L.t_start[t] = a;
                ne = ng = jw = 0;
                w = 0;
            } else if (k == KR_EV_BEGIN_GEN) {  // core.py:200-207
                if (j != ng || j >= L.cap) { fl |= KR_FLAG_LEDGER; continue; }
                sl[4 * j] = a;
                sl[4 * j + 1] = INT64_MIN;  // in flight
                ng++;
            } else if (k == KR_EV_FINISH_GEN) {  // core.py:209-218
                if (j < 0 || j >= ng || sl[4 * j + 1] != INT64_MIN) { fl |= KR_FLAG_LEDGER; continue; }
                sl[4 * j + 1] = a;
            } else if (k == KR_EV_EXEC) {  // core.py:220-229
                if (j != ne || j >= L.cap) { fl |= KR_FLAG_LEDGER; continue; }
                sl[4 * j + 2] = a;
                sl[4 * j + 3] = ev.b[e];
                ne++;
            } else {
                fl |= KR_FLAG_LEDGER;
                continue;
            }
            // waiting.py:81-92, advanced over the newly computable prefix
            while (jw < ne) {
                const int64_t gs = sl[4 * jw], ge = sl[4 * jw + 1];
                const int64_t es = sl[4 * jw + 2], ee = sl[4 * jw + 3];
                int64_t d;
                if (ge - gs >= ee - es) {
                    if (ng <= jw + 1) break;
                    d = sl[4 * (jw + 1)] - ge;
                } else {
                    if (ne <= jw + 1) break;
                    d = sl[4 * (jw + 1) + 2] - ee;
                }
                w += d > 0 ? d : 0;
                jw++;
            }
        }
        L.n_exec[t] = ne;
        L.n_gen[t] = ng;
        L.wait_next[t] = jw;
        L.wait_total[t] = w;
    }
    if (fl && flags) atomicOr(flags, fl);
}
}  // namespace kr

extern "C" int kr_ledger_apply(const kr_ledger* ledger, const kr_events* events, uint32_t* flags,
                               void* stream) {
    if (!ledger || !events || events->n_groups < 0 || ledger->cap < 1) return KR_EINVAL;
    if (events->n_groups == 0) return KR_OK;
    if (!events->task || !events->off || !events->kind || !events->round || !events->a ||
        !events->b)
        return KR_EINVAL;
    k_ledger_apply<<<grid_for(events->n_groups, 128), 128, 0, as_stream(stream)>>>(*ledger, *events,
                                                                                   flags);
    return check_launch("kr_ledger_apply");
}

// ---------------------------------------------------------------------------
// Small planning rounds in one launch (the simulator's per-event plan() call:
// scheduler.py:254-276 over tens to a few thousand pending requests)
// ---------------------------------------------------------------------------
// One CTA: every request's key (urgency_one), a bitonic sort of (key, index)
// pairs in shared memory, and the edge admission (scheduler.py:204-207,
// 223-234: order prefix of length k, stale-observation refetch, skip counter
// reset / increment) -- one launch instead of urgency + select/sort + admit.
// The fleet columns may live in mapped pinned host memory (zero-copy: the
// kernel reads them over PCIe, coalesced), and so may `out` (int32 [3n + 1]:
// order, refetch flag, updated skip counter, validation flags), so a call is
// one launch plus one stream synchronisation.
namespace kr {
constexpr int kPlanSmallMax = 4096;

__device__ __forceinline__ bool pair_less(const kr_key& a, int ia, const kr_key& b, int ib) {
    if (a.hi != b.hi) return a.hi < b.hi;
    if (a.lo != b.lo) return a.lo < b.lo;
    return ia < ib;
}

__global__ void __launch_bounds__(1024) k_plan_small(kr_fleet f, kr_sched c, UrgConst u, int n,
                                                     int P, int k, int32_t* out) {
    extern __shared__ __align__(16) unsigned char sm[];
    kr_key* keys = reinterpret_cast<kr_key*>(sm);
    int* idx = reinterpret_cast<int*>(keys + P);
    __shared__ uint32_t sfl;
    if (threadIdx.x == 0) sfl = 0;
    __syncthreads();
    const FleetSrc s{f};
    const UrgencyOut none{nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                          nullptr};
    uint32_t fl = 0;
    for (int i = threadIdx.x; i < P; i += blockDim.x) {
        kr_key key{~0ull, ~0ull};
        if (i < n) key = urgency_one(s, c, u, none, i, fl);
        keys[i] = key;
        idx[i] = i;
    }
    if (fl) atomicOr(&sfl, fl);
    __syncthreads();
    for (int size = 2; size <= P; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int t = threadIdx.x; t < (P >> 1); t += blockDim.x) {
                const int lo = 2 * t - (t & (stride - 1));
                const int hi = lo + stride;
                const bool up = (lo & size) == 0;
                const kr_key a = keys[lo], b = keys[hi];
                const int ia = idx[lo], ib = idx[hi];
                if (pair_less(b, ib, a, ia) == up) {
                    keys[lo] = b; keys[hi] = a;
                    idx[lo] = ib; idx[hi] = ia;
                }
            }
            __syncthreads();
        }
    }
    for (int p = threadIdx.x; p < n; p += blockDim.x) {
        const int j = idx[p];
        const bool in = p < k;
        out[p] = j;
        out[n + j] = in && (c.now - f.obs_captured_at[j] > c.stale_threshold);
        out[2 * n + j] = in ? 0 : f.skipped[j] + 1;
    }
    __syncthreads();
    if (threadIdx.x == 0) out[3 * n] = static_cast<int32_t>(sfl);
}
}  // namespace kr

extern "C" int kr_plan_small(const kr_fleet* fleet, const kr_sched* cfg, int64_t k, int32_t* out,
                             void* stream) {
    if (!fleet || !cfg || fleet->n < 0 || fleet->n > kPlanSmallMax || k < 0) return KR_EINVAL;
    if (cfg->policy < KR_KAIROS || cfg->policy > KR_LAS || cfg->buckets < 1 ||
        cfg->buckets > 256 || cfg->aging_interval < 1 || cfg->hz_num <= 0 || cfg->hz_den <= 0)
        return KR_EINVAL;
    if (fleet->n == 0) return KR_OK;
    if (!out) return KR_EINVAL;
    const int n = static_cast<int>(fleet->n);
    int P = 1;
    while (P < n) P <<= 1;
    const int threads = P >= 2048 ? 1024 : (P / 2 < 32 ? 32 : P / 2);
    const size_t smem = static_cast<size_t>(P) * (sizeof(kr_key) + sizeof(int));
    if (smem > 48 * 1024) {
        static bool attr = false;
        if (!attr) {
            KR_CUDA_TRY(cudaFuncSetAttribute(k_plan_small, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(kPlanSmallMax * (sizeof(kr_key) + sizeof(int)))));
            attr = true;
        }
    }
    k_plan_small<<<1, threads, smem, as_stream(stream)>>>(*fleet, *cfg, urg_const(*cfg), n, P,
                                                         static_cast<int>(k < n ? k : n), out);
    return check_launch("kr_plan_small");
}

extern "C" int kr_mapped_ptr(void* host, void** device) {
    if (!host || !device) return KR_EINVAL;
    KR_CUDA_TRY(cudaHostGetDevicePointer(device, host, 0));
    return KR_OK;
}
