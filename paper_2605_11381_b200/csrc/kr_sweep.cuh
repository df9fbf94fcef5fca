// kr_sweep.cuh -- threshold sweep / Pareto (horizon.py:135-151, cli.py:104-140):
// C policy configurations decided over the same update magnitudes in one
// streaming pass.  Device code and the per-dtype
// launcher; the C entry point is kr_sweep.cu.
#pragma once
#include <climits>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <type_traits>

#include "kr_common.cuh"
#include "kr_conf.cuh"
#include "kr_host.cuh"
#include "kr_plan.cuh"
#include "kr_stream.cuh"

namespace kr {

// ---------------------------------------------------------------------------
// Threshold sweep (horizon.py:135-151 sweep_thresholds, cli.py:109-140
// cmd_pareto): C policy configurations decided over the same rounds in ONE
// pass over U.
//
// The column statistics (sum, final) do not depend on the configuration, and
// the trip test f > fl(p * m) is monotone in p = 1 + t: with the confidence
// configurations sorted by p, the ones a column trips form a prefix [0, j_n).
// One filter per column gives j_n (fast exits for "none" / "all", otherwise a
// binary search over the sorted factors with the K1 margins, and the
// bit-exact fp64 mean when the margins cannot decide).
//
// A warp owns one robot at a time (lane = VC adjacent columns, chunks of
// 32 * VC columns).  With M_n = max_{n' <= n} j_n' (a warp max-scan carried
// across chunks), configuration c's horizon is the first n with M_n > c, so
// the column where M steps from a to b is the horizon of exactly the
// configurations [a, b) -- one lane per step, no per-configuration loop.  The
// per-configuration sums are accumulated as a difference array over the
// sorted slots (D[a] += n, D[b] -= n; never-tripped slots [M_last, Cc) get
// N), plus a correction F[c] += hmin_c - n for the rare steps below a
// configuration's min_horizon floor.  S_c = prefix_sum(D)[c] + F[c] at the end
// of the CTA; the optional H[c][r] output writes every decision.
// ---------------------------------------------------------------------------
constexpr int kSweepMaxCfg = 64;
constexpr int kSweepPad = 128;  // search tables: a power of two > Cc, padded with +inf
constexpr int kSweepLut = 2048; // ratio buckets

struct SweepCfg {
    int32_t C, Cc;                       // configurations, confidence ones (sorted first)
    int32_t maxcap;                      // max over confidence slots of min(min_horizon, N)
    int32_t half;                        // P / 2: first step of the branch-free search
    int32_t lut_n, lut_shift;            // ratio buckets (0: none), bits dropped per bucket
    uint64_t lut_lo, lut_hi;             // storage-type bit patterns of the bucketed ratio range
    double sfmin, sfmax;                 // column sums whose ratio stays a normal number
    int32_t orig[kSweepMaxCfg];          // sorted slot -> caller's configuration index
    int32_t hcap[kSweepMaxCfg];          // confidence: min(min_horizon, N); static: min(static_h, N)
    double p[kSweepMaxCfg];              // 1 + t, ascending (confidence slots)
    double rh[kSweepPad], rl[kSweepPad]; // ratio bounds (1 + t) / (K - 1) * (1 +/- margin), outward
    uint16_t lut[kSweepLut];             // bucket -> tripping slots, 0xFFFF: undecided
};

// shared copies of the per-configuration tables (indexed per lane)
struct SweepTables {
    double rhd[kSweepPad], rld[kSweepPad];
    float rh[kSweepPad], rl[kSweepPad];
    double p[kSweepMaxCfg];
    int32_t orig[kSweepMaxCfg];
    int32_t hcap[kSweepMaxCfg];
    // per-CTA sums stay below 2^32: R * N elements fit in HBM, so a CTA's share
    // (R / grid robots, N columns, horizons <= N) is < 2^32; checked on the host
    uint32_t D[kSweepMaxCfg + 1];  // difference array of the per-slot sums (mod 2^32)
    uint32_t F[kSweepMaxCfg];      // min_horizon floor corrections
    uint16_t lut[kSweepLut + 2];   // [0]: below the table (0), [lut_n + 1]: above (Cc)
};

// Bit-exact count of tripping confidence configurations for one column.
template <typename T>
__device__ __noinline__ int sweep_exact(const T* col, int K, int N, const double* p, int Cc) {
    const int K1 = K - 1;
    double sum;
    if (N >= 2) {
        sum = to_f64(col[0]);
        for (int k = 1; k < K1; k++) sum = dadd(sum, to_f64(col[static_cast<size_t>(k) * N]));
    } else {
        auto a = [col](int64_t k) { return to_f64(col[k]); };
        sum = np_pairwise_sum(a, 0, K1);
    }
    const double m = ddiv(sum, static_cast<double>(K1));
    const double f = to_f64(col[static_cast<size_t>(K1) * N]);
    int lo = 0, hi = Cc;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (f > dmul(p[mid], m)) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// A warp owns a robot; VC adjacent columns per lane, chunks of 32 VC columns.
// (Measured alternative, not kept: G = 4 / 8 lanes per robot with register-held
// per-lane column blocks cut instructions 2x but the smem-bounded tile leaves
// too few warps per SM -- 36% vs 42% of the HBM peak at C = 16.)
// HALF: two robots per warp (16 lanes x 4 columns, N <= 64 and even).
template <typename T, int KC, int VC, bool HALF = false>
struct SweepWork {
    using CW = ConfWork<T, KC, VC>;
    using Elem = T;
    static constexpr int kVC = VC;
    static constexpr bool kHalf = HALF;
    int K, N, TR, C, Cc, maxcap, half;
    int cw;                      // consumer warps (robots are dealt round-robin to them)
    int lut_n, lut_shift;
    uint64_t lut_lo;
    uint64_t sfminb, sfrng;      // storage-type bits: sums in [sfmin, sfmin + sfrng] filter
    T sfmin, sfmax;
    int32_t* H;                  // [C][R] (nullable)
    unsigned long long* sums;    // [C]
    uint32_t* flags;
    int64_t R;
    // the shared tables sit at a fixed offset of the dynamic shared memory:
    // addressed through the shared window directly (no per-use generic base)
    __device__ __forceinline__ static SweepTables* tables() {
        extern __shared__ __align__(128) unsigned char smem[];
        return reinterpret_cast<SweepTables*>(smem + stream_aux_offset());
    }

    __device__ void setup(int) {}

    // Number of confidence configurations the column trips, or -1 when the
    // margins cannot decide it.  The column's ratio f / sum (one approximate
    // reciprocal) against the slot factors c = (1 + t) / (K - 1): rh[c] / rl[c]
    // widen c by the filter margin (fp32 sum, reciprocal and products:
    // (K + 8) 2^-24; fp64: 2^-49), so ratio > rh[c] is a definite trip and
    // ratio < rl[c] a definite non-trip; both hold for prefixes of the sorted
    // slots.  A bucket table over the ratio's bit pattern answers most columns
    // with one lookup; buckets that straddle a slot bound fall back to a
    // branch-free binary search.  f == 0 never trips; an exact zero mean trips
    // on any f > 0.
    // Branch-free: the bucket lookup (entry 0 / lut_n + 1 stand for the ratios
    // below / above the table) and the zero rules; returns -1 for the columns
    // that need search() (ambiguous bucket, sum out of range).  f == 0 gives
    // ratio bits 0 (below: no trip); sum == 0 < f gives +inf (above: all trip).
    __device__ __forceinline__ int filter(T sf, T fin) const {
        using B = typename std::conditional<sizeof(T) == 4, uint32_t, uint64_t>::type;
        using SB = typename std::make_signed<B>::type;
        B bits, sb;
        if constexpr (sizeof(T) == 4) {
            float r;
            asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(sf));  // <= 1 ulp, sf normal
            bits = __float_as_uint(__fmul_rn(fin, r));
            sb = __float_as_uint(sf);
        } else {
            bits = static_cast<uint64_t>(__double_as_longlong(__dmul_rn(fin, __drcp_rn(sf))));
            sb = static_cast<uint64_t>(__double_as_longlong(sf));
        }
        if (fin == T(0)) bits = 0;
        SB idx = (static_cast<SB>(bits - static_cast<B>(lut_lo)) >> lut_shift) + 1;
        idx = idx < 0 ? 0 : (idx > lut_n + 1 ? lut_n + 1 : idx);
        const int e = tables()->lut[idx];
        const bool out = static_cast<B>(sb - static_cast<B>(sfminb)) > static_cast<B>(sfrng) && sb != 0;
        return e == 0xFFFF || out ? -1 : e;
    }

    __device__ __forceinline__ static T ratio(T sf, T fin) {
        if constexpr (sizeof(T) == 4) {
            float r;
            asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(sf));
            return __fmul_rn(fin, r);
        } else {
            return __dmul_rn(fin, __drcp_rn(sf));
        }
    }

    // ambiguous bucket: branch-free binary search over the slot bounds
    __device__ __forceinline__ int search(T sf, T rho) const {
        if (!(sf >= sfmin && sf <= sfmax)) return -1;
        const T* rh;
        const T* rl;
        if constexpr (sizeof(T) == 4) { rh = tables()->rh; rl = tables()->rl; }
        else { rh = tables()->rhd; rl = tables()->rld; }
        int pos = 0;
        for (int st = half; st > 0; st >>= 1)
            if (rho > rh[pos + st - 1]) pos += st;
        if (pos == Cc || rho < rl[pos]) return pos;
        return -1;
    }

    // configurations [a, b) take horizon n at this robot (a < b)
    __device__ __forceinline__ void step(int a, int b, int n, int64_t r) const {
        atomicAdd(&tables()->D[a], static_cast<uint32_t>(n));
        atomicSub(&tables()->D[b], static_cast<uint32_t>(n));
        if (n < maxcap)  // below some min_horizon floor (horizon.py:130)
            for (int c = a; c < b; c++) {
                const int cap = tables()->hcap[c];
                if (cap > n) atomicAdd(&tables()->F[c], static_cast<uint32_t>(cap - n));
            }
        if (H)
            for (int c = a; c < b; c++) {
                const int cap = tables()->hcap[c];
                H[static_cast<int64_t>(tables()->orig[c]) * R + r] = n > cap ? n : cap;
            }
    }

    __device__ __noinline__ uint32_t check_all(const T* col) const {
        uint32_t fl = 0;
        const int Kr = KC > 0 ? KC : K;
        for (int k = 0; k < Kr; k++)
            for (int c = 0; c < VC; c++) fl |= CW::check(col[k * N + c]);
        return fl;
    }

    // One chunk of 32 VC columns of robot `rob`: trip counts, the warp's
    // max-scan continuing from `carry`, the steps; returns the chunk's
    // running max (the next chunk's carry).
    __device__ __forceinline__ int chunk(const T* rob, int n0c, int carry, int64_t r,
                                         uint32_t& fl) const {
        const int Kr = KC > 0 ? KC : K;
        const int lane = threadIdx.x & 31;
        const int n0 = n0c + lane * VC;
        const bool valid = n0 < N;
        int j[VC];
#pragma unroll
        for (int c = 0; c < VC; c++) j[c] = 0;
        if (valid) {
            const T* col = rob + n0;
            T sf[VC], fin[VC];
            uint32_t mx = 0;
            if constexpr (KC > 0) {
                T x[KC][VC];
#pragma unroll
                for (int k = 0; k < KC; k++) CW::load_row(col + k * N, x[k]);
#pragma unroll
                for (int k = 0; k < KC; k++)
#pragma unroll
                    for (int c = 0; c < VC; c++) mx = max(mx, CW::sexp(x[k][c]));
#pragma unroll
                for (int c = 0; c < VC; c++) {
                    sf[c] = x[0][c];
#pragma unroll
                    for (int k = 1; k < KC - 1; k++) sf[c] = CW::add_rn(sf[c], x[k][c]);
                    fin[c] = x[KC - 1][c];
                }
            } else {
                for (int k = 0; k < Kr; k++) {
                    T x[VC];
                    CW::load_row(col + k * N, x);
#pragma unroll
                    for (int c = 0; c < VC; c++) {
                        mx = max(mx, CW::sexp(x[c]));
                        if (k == 0) sf[c] = x[c];
                        else if (k < Kr - 1) sf[c] = CW::add_rn(sf[c], x[c]);
                        else fin[c] = x[c];
                    }
                }
            }
            const bool bad = mx >= CW::kBad;
            bool any = bad;
#pragma unroll
            for (int c = 0; c < VC; c++) {
                j[c] = filter(sf[c], fin[c]);
                any = any || j[c] < 0;
            }
            if (any) {
                if (bad) fl |= check_all(col);
#pragma unroll
                for (int c = 0; c < VC; c++)
                    if (bad || j[c] < 0) {
                        int jj = bad ? -1 : search(sf[c], ratio(sf[c], fin[c]));
                        if (jj < 0) jj = sweep_exact(col + c, K, N, tables()->p, Cc);
                        j[c] = jj;
                    }
            }
        }
        __syncwarp();
        int jt = carry;
#pragma unroll
        for (int c = 0; c < VC; c++) jt = max(jt, j[c]);
        // inclusive max-scan over the lanes (columns ascend with the lane)
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int o = __shfl_up_sync(0xffffffffu, jt, d);
            if (lane >= d) jt = max(jt, o);
        }
        int cur = __shfl_up_sync(0xffffffffu, jt, 1);
        if (lane == 0) cur = carry;
        if (valid && jt > cur) {
#pragma unroll
            for (int c = 0; c < VC; c++)
                if (j[c] > cur) {
                    step(cur, j[c], n0 + c, r);
                    cur = j[c];
                }
        }
        return __shfl_sync(0xffffffffu, jt, 31);
    }

    // Half-warp robot: lane g of the 16 owns the column pairs 2g, 2g + 1 and
    // 32 + 2g, 33 + 2g (pairs are whole: N is even), so the 16 lanes read each
    // half-row as 128 contiguous bytes (conflict-free 8-byte loads); the max-scan
    // runs over the first 32 columns, then over the second 32 from its total.
    __device__ __forceinline__ static void load_pair(const T* p, T& a, T& b) {
        if constexpr (sizeof(T) == 4) {
            const float2 v = *reinterpret_cast<const float2*>(p);
            a = v.x; b = v.y;
        } else {
            const double2 v = *reinterpret_cast<const double2*>(p);
            a = v.x; b = v.y;
        }
    }

    __device__ __forceinline__ int chunk_half(const T* rob, bool robot_ok, int64_t r,
                                              uint32_t& fl) const {
        const int Kr = KC > 0 ? KC : K;
        const int g = threadIdx.x & 15;
        const int n0 = 2 * g, n1 = 32 + 2 * g;
        const bool p0 = robot_ok && n0 < N, p1 = robot_ok && n1 < N;
        const bool odd = N & 1;  // rows are not pair-aligned: guarded scalar loads
        int j[4] = {0, 0, 0, 0};
        if (p0) {
            T sf[4], fin[4];
            uint32_t mx = 0;
            for (int k = 0; k < Kr; k++) {
                T x[4] = {T(0), T(0), T(0), T(0)};
                const T* row = rob + k * N;
                if (!odd) {
                    load_pair(row + n0, x[0], x[1]);
                    if (p1) load_pair(row + n1, x[2], x[3]);
                } else {  // a column past N stays zero: filter() gives 0
                    x[0] = row[n0];
                    if (n0 + 1 < N) x[1] = row[n0 + 1];
                    if (p1) x[2] = row[n1];
                    if (n1 + 1 < N) x[3] = row[n1 + 1];
                }
#pragma unroll
                for (int c = 0; c < 4; c++) {
                    mx = max(mx, CW::sexp(x[c]));
                    if (k == 0) sf[c] = x[c];
                    else if (k < Kr - 1) sf[c] = CW::add_rn(sf[c], x[c]);
                    else fin[c] = x[c];
                }
            }
            // the padding pair of a lane past N is zeros: filter() gives 0
            const bool bad = mx >= CW::kBad;
            bool any = bad;
#pragma unroll
            for (int c = 0; c < 4; c++) {
                j[c] = filter(sf[c], fin[c]);
                any = any || j[c] < 0;
            }
            if (any) {
                for (int c = 0; c < 4; c++) {
                    const int n = c < 2 ? n0 + c : n1 + c - 2;
                    if (n >= N) continue;
                    const T* col = rob + n;
                    if (bad)
                        for (int k = 0; k < Kr; k++) fl |= CW::check(col[k * N]);
                    if (bad || j[c] < 0) {
                        int jj = bad ? -1 : search(sf[c], ratio(sf[c], fin[c]));
                        if (jj < 0) jj = sweep_exact(col, K, N, tables()->p, Cc);
                        j[c] = jj;
                    }
                }
            }
        }
        __syncwarp();
        int ja = max(j[0], j[1]), jb = max(j[2], j[3]);
#pragma unroll
        for (int d = 1; d < 16; d <<= 1) {  // max-scans within the 16-lane half
            const int oa = __shfl_up_sync(0xffffffffu, ja, d, 16);
            const int ob = __shfl_up_sync(0xffffffffu, jb, d, 16);
            if (g >= d) { ja = max(ja, oa); jb = max(jb, ob); }
        }
        const int ta = __shfl_sync(0xffffffffu, ja, 15, 16);  // M after column 31
        jb = max(jb, ta);
        int ca = __shfl_up_sync(0xffffffffu, ja, 1, 16);
        int cb = __shfl_up_sync(0xffffffffu, jb, 1, 16);
        if (g == 0) { ca = 0; cb = ta; }
        if (p0 && ja > ca) {
            if (j[0] > ca) { step(ca, j[0], n0, r); ca = j[0]; }
            if (j[1] > ca) step(ca, j[1], n0 + 1, r);
        }
        if (p1 && jb > cb) {
            if (j[2] > cb) { step(cb, j[2], n1, r); cb = j[2]; }
            if (j[3] > cb) step(cb, j[3], n1 + 1, r);
        }
        return __shfl_sync(0xffffffffu, jb, 15, 16);
    }

    __device__ __forceinline__ void tile(const TileView& v, int64_t r0, int nr, int) {
        const T* u = reinterpret_cast<const T*>(v.seg[0]);
        uint32_t fl = 0;
        const int Kr = KC > 0 ? KC : K;
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        if (warp >= cw) return;  // the producer warp's slot in the non-TMA modes
        const int KN = Kr * N;
        if constexpr (HALF) {
            const int g = lane & 15;
            for (int rb = warp * 2; rb < nr; rb += cw * 2) {
                const int rr = rb + (lane >> 4);
                const bool ok = rr < nr;
                const int total = chunk_half(u + (ok ? rr : 0) * KN, ok, r0 + rr, fl);
                if (ok && g == 0 && total < Cc) {  // slots never tripped take N
                    atomicAdd(&tables()->D[total], static_cast<uint32_t>(N));
                    if (H)
                        for (int c = total; c < Cc; c++)
                            H[static_cast<int64_t>(tables()->orig[c]) * R + r0 + rr] = N;
                }
                if (ok && H)
                    for (int c = Cc + g; c < C; c += 16)
                        H[static_cast<int64_t>(tables()->orig[c]) * R + r0 + rr] = tables()->hcap[c];
            }
            if (fl && flags) atomicOr(flags, fl);
            return;
        }
        const bool one_chunk = N <= 32 * VC;  // the common shapes (N <= 64 at VC = 2)
        for (int rr = warp; rr < nr; rr += cw) {
            const T* rob = u + rr * KN;
            int carry;
            if (one_chunk) {
                carry = chunk(rob, 0, 0, r0 + rr, fl);
            } else {
                carry = 0;  // M of the previous chunk's last column
                for (int n0c = 0; n0c < N; n0c += 32 * VC) carry = chunk(rob, n0c, carry, r0 + rr, fl);
            }
            // slots never tripped take the whole chunk (>= every floor)
            if (lane == 0 && carry < Cc) {
                atomicAdd(&tables()->D[carry], static_cast<uint32_t>(N));
                if (H)
                    for (int c = carry; c < Cc; c++)
                        H[static_cast<int64_t>(tables()->orig[c]) * R + r0 + rr] = N;
            }
            if (H)
                for (int c = Cc + lane; c < C; c += 32)
                    H[static_cast<int64_t>(tables()->orig[c]) * R + r0 + rr] = tables()->hcap[c];
        }
        if (fl && flags) atomicOr(flags, fl);
    }

    __device__ __forceinline__ void finish(int64_t, int, int, int, int) {}
};

constexpr int kSweepThreads = 384;

template <typename T, int KC, int VC, bool kStaged, bool HALF = false>
__global__ void __launch_bounds__(kSweepThreads, 2) k_horizon_sweep(StreamPlan p,
                                                                         SweepWork<T, KC, VC, HALF> w,
                                                                         const __grid_constant__ SweepCfg cfg) {
    extern __shared__ __align__(128) unsigned char smem[];
    SweepTables* const tab = w.tables();
    for (int i = threadIdx.x; i < w.lut_n; i += blockDim.x) tab->lut[i + 1] = cfg.lut[i];
    if (threadIdx.x == 0) {
        tab->lut[0] = 0;
        tab->lut[w.lut_n + 1] = static_cast<uint16_t>(w.Cc);
    }
    for (int i = threadIdx.x; i < kSweepPad; i += blockDim.x) {
        tab->rhd[i] = cfg.rh[i];
        tab->rld[i] = cfg.rl[i];
        tab->rh[i] = static_cast<float>(cfg.rh[i]);  // exactly representable (host-rounded)
        tab->rl[i] = static_cast<float>(cfg.rl[i]);
        if (i < kSweepMaxCfg) {
            tab->p[i] = cfg.p[i];
            tab->orig[i] = cfg.orig[i];
            tab->hcap[i] = cfg.hcap[i];
            tab->F[i] = 0;
        }
        if (i <= kSweepMaxCfg) tab->D[i] = 0;
    }
    __syncthreads();
    stream_run<kStaged>(p, smem, w);
    __syncthreads();
    if (threadIdx.x == 0) {  // S_c = prefix_sum(D)[c] + F[c]; static slots once per grid
        uint32_t run = 0;
        for (int c = 0; c < w.Cc; c++) {
            run += tab->D[c];
            const uint32_t s = run + tab->F[c];
            if (s) atomicAdd(&w.sums[tab->orig[c]], static_cast<unsigned long long>(s));
        }
        if (blockIdx.x == 0)
            for (int c = w.Cc; c < w.C; c++)
                atomicAdd(&w.sums[tab->orig[c]],
                          static_cast<unsigned long long>(w.R) * static_cast<unsigned long long>(tab->hcap[c]));
    }
}


// Launch of the per-dtype sweep kernels (instantiated in kr_sweep_f32.cu /
// kr_sweep_f64.cu so the two halves compile in parallel).
template <typename T>
int sweep_run(const void* U, int64_t R, int32_t K, int32_t N, int32_t C, int32_t Cc,
              const SweepCfg& cfg, unsigned long long* sums, int32_t* H, uint32_t* flags,
              cudaStream_t st) {
    uint64_t rb = static_cast<uint64_t>(K) * N * sizeof(T);
    const void* bases[1] = {U};
    auto go = [&](auto proto, auto kstaged, auto kdirect) -> int {
        using W = decltype(proto);
        // a warp per robot (32 "items"): 11 consumer warps x 2 robots per tile,
        // two CTAs (24 warps) per SM -- the per-robot scan is instruction-heavy,
        // so warps, not bytes in flight, set the pace
        StreamPlan p = make_plan(1, bases, &rb, R, W::kHalf ? 16 : 32, 0, kSweepThreads - 32,
                                 kernel_regs(kstaged), 2,
                                 static_cast<uint32_t>(sizeof(SweepTables)), W::kHalf ? 44 : 22);
        // per-CTA 32-bit sums: robots per CTA (grid >= SMs) x N < 2^32
        if ((R / device_info().sm_count + 1) * static_cast<int64_t>(N) >= (int64_t(1) << 32))
            return KR_EINVAL;
        W w{};
        w.K = K; w.N = N; w.TR = p.TR; w.C = C; w.Cc = Cc; w.maxcap = cfg.maxcap;
        w.half = cfg.half;
        w.cw = p.threads / 32;
        w.sfmin = static_cast<T>(cfg.sfmin);
        w.sfmax = static_cast<T>(cfg.sfmax);
        w.lut_n = cfg.lut_n; w.lut_shift = cfg.lut_shift; w.lut_lo = cfg.lut_lo;
        if (cfg.sfmin <= cfg.sfmax) {
            uint64_t lo, hi;
            if constexpr (sizeof(T) == 4) {
                const float a = static_cast<float>(cfg.sfmin), b = static_cast<float>(cfg.sfmax);
                uint32_t ua, ub;
                std::memcpy(&ua, &a, 4); std::memcpy(&ub, &b, 4);
                lo = ua; hi = ub;
            } else {
                std::memcpy(&lo, &cfg.sfmin, 8); std::memcpy(&hi, &cfg.sfmax, 8);
            }
            w.sfminb = lo; w.sfrng = hi - lo;
        } else {  // no sum filters (every nonzero sum is searched / exact)
            w.sfminb = 0; w.sfrng = 0;
        }
        w.H = H; w.sums = sums; w.flags = flags; w.R = R;
        return launch_stream(kstaged, kdirect, p, w, st, "kr_horizon_sweep", 0, cfg);
    };
    // N > 64 (or a misaligned base): a warp per robot, chunks of 32 lanes x VC
    // columns; VC = 2 (pair loads) when the rows allow it.  (VC = 4 was
    // measured 2x slower at N = 128: 0.86 vs 1.75 ms, register spills.)
    const bool al = (reinterpret_cast<uintptr_t>(U) & 15u) == 0;
#define KR_SWEEP(KK, VV) \
    return go(SweepWork<T, KK, VV>{}, k_horizon_sweep<T, KK, VV, true>, k_horizon_sweep<T, KK, VV, false>)
    // two robots per warp: N <= 64 (pair loads when N is even and the base 16-byte aligned)
    static const bool half_off = std::getenv("KR_SWEEP_NO_HALF") != nullptr;  // A/B knob
    if (!half_off && N <= 64 && (N % 2 == 1 || al)) {
        if (K == 6)
            return go(SweepWork<T, 6, 1, true>{}, k_horizon_sweep<T, 6, 1, true, true>,
                      k_horizon_sweep<T, 6, 1, false, true>);
        return go(SweepWork<T, 0, 1, true>{}, k_horizon_sweep<T, 0, 1, true, true>,
                  k_horizon_sweep<T, 0, 1, false, true>);
    }
    if (al && N % 2 == 0 && N > 32) {
        if (K == 6) KR_SWEEP(6, 2);
        KR_SWEEP(0, 2);
    }
    KR_SWEEP(0, 1);
#undef KR_SWEEP
}

int sweep_run_f32(const void* U, int64_t R, int32_t K, int32_t N, int32_t C, int32_t Cc,
                  const SweepCfg& cfg, unsigned long long* sums, int32_t* H, uint32_t* flags,
                  cudaStream_t st);
int sweep_run_f64(const void* U, int64_t R, int32_t K, int32_t N, int32_t C, int32_t Cc,
                  const SweepCfg& cfg, unsigned long long* sums, int32_t* H, uint32_t* flags,
                  cudaStream_t st);

}  // namespace kr
