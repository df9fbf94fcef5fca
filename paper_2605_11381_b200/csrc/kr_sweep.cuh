// kr_sweep.cuh -- threshold sweep / Pareto (horizon.py:135-151, cli.py:104-140):
// C policy configurations decided over the same update magnitudes in one
// streaming pass.  Device code and the per-dtype
// launcher; the C entry point is kr_sweep.cu.
#pragma once
#include <algorithm>
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
// Two layouts: the segmented kernel (SweepSeg, below: G lanes per robot, each
// deciding a register-resident window of columns) for 16 <= N <= 512 where
// its windows do not collide in shared-memory banks, and otherwise the
// warp-per-robot kernel (SweepWork): a warp owns one robot at a time (lane =
// VC adjacent columns, chunks of 32 * VC columns).  With M_n = max_{n' <= n} j_n' (a warp max-scan carried
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
    alignas(16) int32_t orig[kSweepMaxCfg];  // sorted slot -> caller's configuration index
    alignas(16) int32_t hcap[kSweepMaxCfg];  // confidence: min(min_horizon, N); static: min(static_h, N)
    alignas(16) double p[kSweepMaxCfg];      // 1 + t, ascending (confidence slots)
    alignas(16) double rh[kSweepPad];        // ratio bounds (1 + t) / (K - 1) * (1 +/- margin),
    alignas(16) double rl[kSweepPad];        //   outward
    alignas(16) uint16_t lut[kSweepLut]; // bucket -> tripping slots, 0xFFFF: undecided
    uint64_t clamp_base;                 // bits of clamp_lo (segmented kernel's table origin)
    double clamp_lo, clamp_hi;           // ratio clamp: the below / above entries
    uint16_t lut_below, lut_above;       // sentinel entries (0 / Cc; 0xFFFF without a table)
};

// shared copies of the per-configuration tables (indexed per lane)
struct SweepTables {
    alignas(16) double rhd[kSweepPad];
    alignas(16) double rld[kSweepPad];
    alignas(16) double p[kSweepMaxCfg];
    alignas(16) int32_t orig[kSweepMaxCfg];
    alignas(16) int32_t hcap[kSweepMaxCfg];
    float rh[kSweepPad], rl[kSweepPad];
    // per-CTA sums stay below 2^32: R * N elements fit in HBM, so a CTA's share
    // (R / grid robots, N columns, horizons <= N) is < 2^32; checked on the host
    uint32_t D[kSweepMaxCfg + 1];  // difference array of the per-slot sums (mod 2^32)
    uint32_t F[kSweepMaxCfg];      // min_horizon floor corrections
    // bucket table: entries at [kLutBase, kLutBase + lut_n) (16-byte aligned for
    // the vector copy), [kLutBase - 1]: below the table (0), [kLutBase + lut_n]:
    // above (Cc)
    alignas(16) uint16_t lut[kSweepLut + 16];
};
constexpr int kLutBase = 8;

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
        SB idx = (static_cast<SB>(bits - static_cast<B>(lut_lo)) >> lut_shift) + kLutBase;
        idx = idx < kLutBase - 1 ? kLutBase - 1 : (idx > lut_n + kLutBase ? lut_n + kLutBase : idx);
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
        int j[4] = {0, 0, 0, 0};
        if (p0) {
            T sf[4], fin[4];
            uint32_t mx = 0;
            if (!(N & 1)) {
                // even N: straight-line pair loads; a lane without a second pair
                // re-reads its first one (already validated, its trips masked below)
                const int n1c = p1 ? n1 : n0;
                auto row = [&](int k) {
                    T x[4];
                    load_pair(rob + k * N + n0, x[0], x[1]);
                    load_pair(rob + k * N + n1c, x[2], x[3]);
#pragma unroll
                    for (int c = 0; c < 4; c++) {
                        mx = max(mx, CW::sexp(x[c]));
                        if (k == 0) sf[c] = x[c];
                        else if (k < Kr - 1) sf[c] = CW::add_rn(sf[c], x[c]);
                        else fin[c] = x[c];
                    }
                };
                if constexpr (KC > 0) {
#pragma unroll
                    for (int k = 0; k < KC; k++) row(k);
                } else {
                    for (int k = 0; k < Kr; k++) row(k);
                }
            } else {  // odd N: rows are not pair-aligned; a column past N stays zero
                for (int k = 0; k < Kr; k++) {
                    T x[4] = {T(0), T(0), T(0), T(0)};
                    const T* row = rob + k * N;
                    x[0] = row[n0];
                    if (n0 + 1 < N) x[1] = row[n0 + 1];
                    if (p1) x[2] = row[n1];
                    if (n1 + 1 < N) x[3] = row[n1 + 1];
#pragma unroll
                    for (int c = 0; c < 4; c++) {
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
            for (int c = 0; c < 4; c++) {
                j[c] = filter(sf[c], fin[c]);
                if (c >= 2 && !p1) j[c] = 0;  // no second pair (odd N: zeros filter to 0)
                any = any || j[c] < 0;
            }
            if (any) {
#pragma unroll
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

// ---------------------------------------------------------------------------
// Segmented sweep (the default for N <= 512): G lanes per robot, each lane
// owning a window of CPL (14 or 16) columns (VW = 2: column pairs with
// 8/16-byte loads), 32 / G robots per warp.  Pass 1 decides every column of
// the segment in registers with no cross-lane traffic: K row loads, the
// validation max, the fp32 sums (packed FADD2 for pairs), and the bucket-table
// lookup on the CLAMPED ratio -- clamping the ratio to the table's range
// replaces the index clamp and the zero rules (f == 0: ratio 0 or NaN -> the
// "below" entry, no trip; sum == 0 < f: +inf -> the "above" entry, all trip).
// The per-lane range checks fold into two reductions: the element maximum
// bounds every column sum from above, and an unsigned minimum over
// bits(sum) - 1 (a zero sum wraps to the top) bounds them from below.  Pass 2
// is one exclusive max-scan over the robot's G segment maxima; only a lane
// whose segment raises the running maximum walks its registers for the steps.
// Columns the table cannot decide (and invalid or out-of-range lanes) are
// re-decided one by one in sweep_fix, off the straight-line path.
// Lane mapping q = lane % (32 / G) (robot), s = lane / (32 / G) (segment):
// for N = 50 fp32 the 8-byte row loads of a half-warp hit 16 distinct bank
// pairs (robot stride 300 words = 12 mod 32 banks, segment stride 14).
// ---------------------------------------------------------------------------
constexpr int kSegCols = 16;  // columns per lane (compile-time register array)

// One column re-decided exactly (rare path): (flags << 16) | trip count.
template <typename T, int KC>
__device__ __noinline__ int sweep_fix(const T* col, int K, int N, int jf, bool check_vals,
                                      T sfmin, T sfmax, int half, int Cc, const double* p,
                                      const T* rh, const T* rl) {
    using CW = ConfWork<T, KC, 1>;
    const int Kr = KC > 0 ? KC : K;
    uint32_t fl = 0, mx = 0;
    T sf = col[0], fin = col[static_cast<size_t>(Kr - 1) * N];
    for (int k = 0; k < Kr; k++) {
        const T x = col[static_cast<size_t>(k) * N];
        mx = max(mx, CW::sexp(x));
        if (check_vals) fl |= CW::check(x);
        if (k >= 1 && k < Kr - 1) sf = CW::add_rn(sf, x);
    }
    const bool colbad = mx >= CW::kBad;
    const bool inr = sf == T(0) || (sf >= sfmin && sf <= sfmax);
    int j = jf;
    if (colbad || !inr || jf == 0xFFFF) {
        j = -1;
        if (!colbad && sf >= sfmin && sf <= sfmax) {  // branch-free binary search
            T rho;
            if constexpr (sizeof(T) == 4) {
                float r;
                asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(sf));
                rho = __fmul_rn(fin, r);
            } else {
                rho = __dmul_rn(fin, __drcp_rn(sf));
            }
            int pos = 0;
            for (int st = half; st > 0; st >>= 1)
                if (rho > rh[pos + st - 1]) pos += st;
            if (pos == Cc || rho < rl[pos]) j = pos;
        }
        if (j < 0) j = sweep_exact(col, K, N, p, Cc);
    }
    return static_cast<int>(fl << 16) | j;
}

template <typename T, int KC, int VW, int CPL, bool ROT = false>
struct SweepSeg {
    using CW = ConfWork<T, KC, 1>;
    using B = typename std::conditional<sizeof(T) == 4, uint32_t, uint64_t>::type;
    using Elem = T;
    static constexpr int kVC = VW;
    static constexpr bool kRot = ROT;
    int K, N, C, Cc, maxcap, half;
    int G, RW, lgRW;             // lanes per robot, robots per warp (32 / G), log2(RW)
    int cw;                      // consumer warps
    int lut_shift;
    B lut_base;                  // bits of clo: table index = (bits(rho) - lut_base) >> lut_shift
    T clo, chi;                  // ratio clamp: the "below" / "above" entries
    uint32_t emaxb;              // element bound (sexp) keeping every sum <= sfmax
    B sfminb1;                   // bits(sfmin) - 1
    T sfmin, sfmax;
    int32_t* H;                  // [C][R] (nullable)
    unsigned long long* sums;    // [C]
    uint32_t* flags;
    int64_t R;
    __device__ __forceinline__ static SweepTables* tables() {
        extern __shared__ __align__(128) unsigned char smem[];
        return reinterpret_cast<SweepTables*>(smem + stream_aux_offset());
    }
    __device__ void setup(int) {}
    // per-warp task list of the cooperative exact path (32 x CPL entries)
    __device__ __forceinline__ static uint16_t* fix_tasks(int warp) {
        extern __shared__ __align__(128) unsigned char smem[];
        return reinterpret_cast<uint16_t*>(smem + stream_aux_offset() + sizeof(SweepTables)) +
               warp * 32 * kSegCols;
    }

    __device__ __forceinline__ static B bits_of(T x) {
        if constexpr (sizeof(T) == 4) return __float_as_uint(x);
        else return static_cast<uint64_t>(__double_as_longlong(x));
    }

    // trip count of one column from its sum and final magnitude (bucket table)
    __device__ __forceinline__ int lookup(T sf, T fin, B& mn) const {
        T rho;
        if constexpr (sizeof(T) == 4) {
            float r;
            asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(sf));  // <= 1 ulp, sf normal
            rho = fminf(fmaxf(__fmul_rn(fin, r), clo), chi);
        } else {
            rho = fmin(fmax(__dmul_rn(fin, __drcp_rn(sf)), clo), chi);
        }
        mn = min(mn, bits_of(sf) - B(1));
        const uint32_t idx = static_cast<uint32_t>((bits_of(rho) - lut_base) >> lut_shift);
        return (tables()->lut + (kLutBase - 1))[idx];  // [0]: below, [lut_n + 1]: above
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

    // byte i of the packed running maxima
    __device__ __forceinline__ static int byte_at(const uint32_t (&pk)[(CPL + 3) / 4], int i) {
        uint32_t w = pk[0];
#pragma unroll
        for (int t = 1; t < (CPL + 3) / 4; t++) w = (i >> 2) == t ? pk[t] : w;
        return static_cast<int>((w >> ((i & 3) * 8)) & 0xFFu);
    }

    __device__ __forceinline__ void tile(const TileView& v, int64_t r0, int nr, int) {
        const T* u = reinterpret_cast<const T*>(v.seg[0]);
        const int Kr = KC > 0 ? KC : K;
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        if (warp >= cw) return;
        const int q = lane & (RW - 1), sg = lane >> lgRW;
        const int KN = Kr * N;
        // the lane's window of CPL columns; the last windows are shifted left to
        // end at N (their leading columns repeat the previous lane's: those are
        // below the scan's carry, so they never step twice)
        const int c0 = min(sg * CPL, N - CPL);
        // ROT (robot strides that are multiples of 32 banks, e.g. N = 64 / 128
        // fp32): lane (q, s) walks its window's column groups rotated by
        // q + RW (s / 2), so the lanes of a phase read distinct banks; j[i]
        // then holds column colof(i), and pass 2 restores column order
        constexpr int kP = CPL / VW;
        static_assert(!ROT || (kP & (kP - 1)) == 0, "rotation needs a power-of-two group count");
        const int rot = ROT ? ((q + RW * (sg >> 1)) & (kP - 1)) : 0;
        auto colof = [&](int i) { return ROT ? VW * (((i / VW) + rot) & (kP - 1)) + i % VW : i; };
        uint32_t fl = 0;
        for (int rb = warp * RW; rb < nr; rb += cw * RW) {
            const int rr = rb + q;
            const bool ok = rr < nr;
            const T* rob = u + (ok ? rr : 0) * KN;  // lanes past the tile re-read robot 0
            const T* base = rob + c0;
            int j[CPL];
            uint32_t mx = 0;
            B mn = ~B(0);
            int m = 0;
            if constexpr (VW == 2 && sizeof(T) == 4) {
                // row pointers once per robot: every pair load below is [row + imm]
                const T* rowp[KC > 0 ? KC : 1];
                if constexpr (KC > 0) {
#pragma unroll
                    for (int k = 0; k < KC; k++) rowp[k] = base + k * N;
                }
#pragma unroll
                for (int i = 0; i < CPL; i += 2) {
                    float2 x, sf;
                    auto ld = [&](int k) {
                        const T* rp = KC > 0 ? rowp[KC > 0 ? k : 0] : base + k * N;
                        x = *reinterpret_cast<const float2*>(rp + colof(i));
                        mx = max(mx, max(__float_as_uint(x.x), __float_as_uint(x.y)));
                    };
                    auto add2 = [&]() {
                        unsigned long long a2, b2, o2;
                        memcpy(&a2, &sf, 8);
                        memcpy(&b2, &x, 8);
                        asm("add.rn.f32x2 %0, %1, %2;" : "=l"(o2) : "l"(a2), "l"(b2));
                        memcpy(&sf, &o2, 8);
                    };
                    ld(0);
                    sf = x;
                    if constexpr (KC > 0) {
#pragma unroll
                        for (int k = 1; k < KC - 1; k++) { ld(k); add2(); }
                        ld(KC - 1);
                    } else {
                        for (int k = 1; k < Kr - 1; k++) { ld(k); add2(); }
                        ld(Kr - 1);
                    }
                    j[i] = lookup(sf.x, x.x, mn);
                    j[i + 1] = lookup(sf.y, x.y, mn);
                    m = max(m, max(j[i], j[i + 1]));
                }
            } else {
                const T* rowp[KC > 0 ? KC : 1];
                if constexpr (KC > 0) {
#pragma unroll
                    for (int k = 0; k < KC; k++) rowp[k] = base + k * N;
                }
#pragma unroll
                for (int i = 0; i < CPL; i += VW) {
                    T sf[VW], x[VW];
                    auto ldv = [&](int k) {  // VW adjacent columns of row k
                        const T* rp = (KC > 0 ? rowp[KC > 0 ? k : 0] : base + k * N) + colof(i);
                        if constexpr (VW == 2 && sizeof(T) == 8) {
                            const double2 d = *reinterpret_cast<const double2*>(rp);
                            x[0] = d.x;
                            x[VW - 1] = d.y;
                        } else {
#pragma unroll
                            for (int c = 0; c < VW; c++) x[c] = rp[c];
                        }
                    };
                    ldv(0);
#pragma unroll
                    for (int c = 0; c < VW; c++) {
                        sf[c] = x[c];
                        mx = max(mx, CW::sexp(x[c]));
                    }
                    auto rowk = [&](int k, bool add) {
                        ldv(k);
#pragma unroll
                        for (int c = 0; c < VW; c++) {
                            mx = max(mx, CW::sexp(x[c]));
                            if (add) sf[c] = CW::add_rn(sf[c], x[c]);
                        }
                    };
                    if constexpr (KC > 0) {
#pragma unroll
                        for (int k = 1; k < KC; k++) rowk(k, k < KC - 1);
                    } else {
                        for (int k = 1; k < Kr; k++) rowk(k, k < Kr - 1);
                    }
#pragma unroll
                    for (int c = 0; c < VW; c++) {
                        j[i + c] = lookup(sf[c], x[c], mn);
                        m = max(m, j[i + c]);
                    }
                }
            }
            // rare: undecided buckets, invalid values, sums outside [sfmin, sfmax].
            // The warp's columns that need an exact decision are dealt to all 32
            // lanes (undecided columns cluster in the tail windows: one lane
            // would otherwise run them one after another).
            const bool need = ok && (mx > emaxb || mn < sfminb1 || m >= 0xFFFF);
            if (__any_sync(0xffffffffu, need)) {
                const bool all = mx > emaxb || mn < sfminb1;  // re-check every column
                uint32_t fm = 0;
                if (need) {
#pragma unroll
                    for (int i = 0; i < CPL; i++)
                        if (all || j[i] == 0xFFFF) fm |= 1u << i;
                }
                const int cnt = __popc(fm);
                int inc = cnt;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const int o = __shfl_up_sync(0xffffffffu, inc, d);
                    if (lane >= d) inc += o;
                }
                const int total = __shfl_sync(0xffffffffu, inc, 31);
                uint16_t* task = fix_tasks(warp);
                {
                    const uint32_t chk = mx >= CW::kBad ? 1u : 0u;
                    uint32_t f = fm;
                    int o = inc - cnt;
                    while (f) {
                        const int i = __ffs(f) - 1;
                        f &= f - 1;
                        task[o++] = static_cast<uint16_t>(i | (lane << 4) | (chk << 9));
                    }
                }
                __syncwarp();
                const T* rh = sizeof(T) == 4 ? reinterpret_cast<const T*>(tables()->rh)
                                             : reinterpret_cast<const T*>(tables()->rhd);
                const T* rl = sizeof(T) == 4 ? reinterpret_cast<const T*>(tables()->rl)
                                             : reinterpret_cast<const T*>(tables()->rld);
                for (int t = lane; t < total; t += 32) {
                    const uint32_t e = task[t];
                    const int L = (e >> 4) & 31;
                    int ci = static_cast<int>(e & 15);
                    if constexpr (ROT) {  // the owner's rotation
                        const int rL = ((L & (RW - 1)) + RW * ((L >> lgRW) >> 1)) & (kP - 1);
                        ci = VW * (((ci / VW) + rL) & (kP - 1)) + ci % VW;
                    }
                    const int cL = min((L >> lgRW) * CPL, N - CPL) + ci;
                    const T* col = u + (rb + (L & (RW - 1))) * KN + cL;
                    const int pk = sweep_fix<T, KC>(col, K, N, 0xFFFF, (e >> 9) & 1, sfmin, sfmax,
                                                    half, Cc, tables()->p, rh, rl);
                    task[t] = static_cast<uint16_t>((pk & 0xFF) | ((static_cast<uint32_t>(pk) >> 16) << 8));
                }
                __syncwarp();
                if (fm) {
                    int o = inc - cnt;
                    m = 0;
#pragma unroll
                    for (int i = 0; i < CPL; i++) {
                        if ((fm >> i) & 1u) {
                            const uint32_t e = task[o++];
                            j[i] = static_cast<int>(e & 0xFF);
                            fl |= e >> 8;
                        }
                        m = max(m, j[i]);
                    }
                }
                __syncwarp();  // the task list is rewritten by the next robot group
            }
            // exclusive max-scan over the robot's segments (lanes q, q + RW, ...)
            int vv = m;
            for (int d = 1; d < G; d <<= 1) {
                const int o = __shfl_up_sync(0xffffffffu, vv, d * RW);
                if (sg >= d) vv = max(vv, o);
            }
            int cur = __shfl_up_sync(0xffffffffu, vv, RW);
            if (sg == 0) cur = 0;
            const int64_t r = r0 + rr;
            if (ok && m > cur) {  // this segment raises the running maximum
                if constexpr (ROT) {  // column order through this lane's task-list row
                    uint16_t* sc = fix_tasks(warp) + lane * kSegCols;
#pragma unroll
                    for (int i = 0; i < CPL; i++) sc[colof(i)] = static_cast<uint16_t>(j[i]);
#pragma unroll
                    for (int i = 0; i < CPL; i++) j[i] = sc[i];
                }
                // branch-free: the columns where it rises, and the running maxima
                uint32_t mask = 0;
                uint32_t pk[(CPL + 3) / 4];
                int run = cur;
#pragma unroll
                for (int i = 0; i < CPL; i++) {
                    if (j[i] > run) mask |= 1u << i;
                    run = max(run, j[i]);
                    if ((i & 3) == 0) pk[i >> 2] = static_cast<uint32_t>(run);
                    else pk[i >> 2] |= static_cast<uint32_t>(run) << ((i & 3) * 8);
                }
                int a2 = cur;
                while (mask) {
                    const int i = __ffs(mask) - 1;
                    mask &= mask - 1;
                    const int b2 = byte_at(pk, i);
                    step(a2, b2, c0 + i, r);
                    a2 = b2;
                }
            }
            if (ok && sg == G - 1 && vv < Cc) {  // slots never tripped take N
                atomicAdd(&tables()->D[vv], static_cast<uint32_t>(N));
                if (H)
                    for (int c = vv; c < Cc; c++)
                        H[static_cast<int64_t>(tables()->orig[c]) * R + r] = N;
            }
            if (ok && H)
                for (int c = Cc + sg; c < C; c += G)
                    H[static_cast<int64_t>(tables()->orig[c]) * R + r] = tables()->hcap[c];
        }
        if (fl && flags) atomicOr(flags, fl);
    }

    __device__ __forceinline__ void finish(int64_t, int, int, int, int) {}
};

constexpr int kSweepThreads = 384;

// n16 16-byte pieces from the (16-byte aligned) parameter space to shared memory.
__device__ __forceinline__ void param_copy16(void* dst, const void* src, int n16) {
    const uint4* s = reinterpret_cast<const uint4*>(src);
    uint4* d = reinterpret_cast<uint4*>(dst);
    for (int i = threadIdx.x; i < n16; i += blockDim.x) d[i] = s[i];
}

// Shared tables from the parameter space, in 16-byte pieces: a load whose
// address differs across the warp is issued once per distinct address, so
// wide pieces (not 2- or 8-byte elements) keep the prologue short.
__device__ __forceinline__ void sweep_prologue(SweepTables* tab, const SweepCfg& cfg) {
    param_copy16(tab->lut + kLutBase, cfg.lut, (cfg.lut_n * 2 + 15) / 16);
    param_copy16(tab->rhd, cfg.rh, kSweepPad * 8 / 16);
    param_copy16(tab->rld, cfg.rl, kSweepPad * 8 / 16);
    param_copy16(tab->p, cfg.p, kSweepMaxCfg * 8 / 16);
    param_copy16(tab->orig, cfg.orig, kSweepMaxCfg * 4 / 16);
    param_copy16(tab->hcap, cfg.hcap, kSweepMaxCfg * 4 / 16);
    if (threadIdx.x == 0) {
        tab->lut[kLutBase - 1] = cfg.lut_below;
        tab->lut[kLutBase + cfg.lut_n] = cfg.lut_above;
    }
    for (int i = threadIdx.x; i <= kSweepMaxCfg; i += blockDim.x) {
        tab->D[i] = 0;
        if (i < kSweepMaxCfg) tab->F[i] = 0;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kSweepPad; i += blockDim.x) {
        tab->rh[i] = static_cast<float>(tab->rhd[i]);  // exactly representable (host-rounded)
        tab->rl[i] = static_cast<float>(tab->rld[i]);
    }
    __syncthreads();
}

// S_c = prefix_sum(D)[c] + F[c] per CTA; static slots once per grid
__device__ __forceinline__ void sweep_epilogue(const SweepTables* tab, int Cc, int C, int64_t R,
                                               unsigned long long* sums) {
    __syncthreads();
    if (threadIdx.x == 0 && sums) {  // (no sums: a decide-only launch, H is the output)
        uint32_t run = 0;
        for (int c = 0; c < Cc; c++) {
            run += tab->D[c];
            const uint32_t s = run + tab->F[c];
            if (s) atomicAdd(&sums[tab->orig[c]], static_cast<unsigned long long>(s));
        }
        if (blockIdx.x == 0)
            for (int c = Cc; c < C; c++)
                atomicAdd(&sums[tab->orig[c]],
                          static_cast<unsigned long long>(R) * static_cast<unsigned long long>(tab->hcap[c]));
    }
}

template <typename T, int KC, int VC, bool kStaged, bool HALF = false>
__global__ void __launch_bounds__(kSweepThreads, 2) k_horizon_sweep(StreamPlan p,
                                                                         SweepWork<T, KC, VC, HALF> w,
                                                                         const __grid_constant__ SweepCfg cfg) {
    extern __shared__ __align__(128) unsigned char smem[];
    SweepTables* const tab = w.tables();
    sweep_prologue(tab, cfg);
    stream_run<kStaged>(p, smem, w);
    sweep_epilogue(tab, w.Cc, w.C, w.R, w.sums);
}

// Register budget.  LEAN (decide-only launches of the fp32 pair kernel, i.e.
// confidence horizons beside the planning round's side stream) is held to 80
// registers (__launch_bounds__(384, 2)): 128 measured 1% faster alone, but 80
// leaves room on every SM for the side stream (urgency: 2 CTAs of 256 threads
// at 64 registers beside the two decide CTAs), confidence round 266 -> 258 us
// (profiles/r2_confidence_layouts.jsonl).  Sweeps keep 128: at 80 the exact
// path spills (tie-heavy sweep 0.67 -> 0.79 ms, fp64 0.49 -> 0.59 ms).
template <bool LEAN>
struct SegBounds {
    static constexpr int kThreads = LEAN ? 384 : 512;
    static constexpr int kMinBlocks = LEAN ? 2 : 1;
};
constexpr int kSegThreads = 384;  // largest CTA the launcher plans (<= both bounds)

template <typename T, int KC, int VW, bool kStaged>
__global__ void __launch_bounds__(512, 1)
k_horizon_sweep_seg_rot(StreamPlan p, SweepSeg<T, KC, VW, 16, true> w, const __grid_constant__ SweepCfg cfg) {
    extern __shared__ __align__(128) unsigned char smem[];
    SweepTables* const tab = w.tables();
    sweep_prologue(tab, cfg);
    stream_run<kStaged>(p, smem, w);
    sweep_epilogue(tab, w.Cc, w.C, w.R, w.sums);
}

template <typename T, int KC, int VW, int CPL, bool kStaged, bool LEAN = false>
__global__ void __launch_bounds__(SegBounds<LEAN>::kThreads, SegBounds<LEAN>::kMinBlocks)
k_horizon_sweep_seg(StreamPlan p, SweepSeg<T, KC, VW, CPL> w,
                                                                    const __grid_constant__ SweepCfg cfg) {
    extern __shared__ __align__(128) unsigned char smem[];
    SweepTables* const tab = w.tables();
    sweep_prologue(tab, cfg);
    stream_run<kStaged>(p, smem, w);
    sweep_epilogue(tab, w.Cc, w.C, w.R, w.sums);
}


// Shared-memory wavefronts of the segmented kernel's first row load (lane q =
// lane % RW reads robot q, window c0(s)): the robot stride in banks decides
// whether the windows of a phase collide (N = 50 fp32: 1, conflict-free;
// N = 64 / 128 fp32: every robot on the same banks).  Above 2 the launcher
// keeps the warp-per-robot kernels.
inline int sweep_seg_conflicts(int K, int N, size_t es, bool pair, bool rot = false) {
    int G = 1;
    while (G * kSegCols < N) G <<= 1;
    const int CPL = rot ? kSegCols : (pair && G * 14 >= N ? 14 : kSegCols);
    const int VWc = pair ? 2 : 1, P = CPL / VWc;
    const int RW = 32 / G;
    const int w = static_cast<int>(es / 4);         // words per element
    const int width = (pair ? 2 : 1) * w;           // words per lane access
    const int lanes = width >= 4 ? 8 : (width == 2 ? 16 : 32);  // lanes per phase
    int worst = 1;
    for (int ph = 0; ph < 32; ph += lanes) {
        long words[32][32];  // per bank: the distinct words the phase touches
        int cnt[32] = {};
        for (int l = ph; l < ph + lanes; l++) {
            const int q = l % RW, sg = l / RW;
            const int c0 = std::min(sg * CPL, N - CPL) + (rot ? VWc * ((q + RW * (sg >> 1)) % P) : 0);
            const long a0 = (static_cast<long>(q) * K * N + c0) * w;
            for (int t = 0; t < width; t++) {
                const long wd = a0 + t;
                const int b = static_cast<int>(wd & 31);
                bool seen = false;
                for (int z = 0; z < cnt[b]; z++) seen = seen || words[b][z] == wd;
                if (!seen) words[b][cnt[b]++] = wd;
            }
        }
        for (int b = 0; b < 32; b++) worst = std::max(worst, cnt[b]);
    }
    return worst;
}

// Launch of the per-dtype sweep kernels (instantiated in kr_sweep_f32.cu /
// kr_sweep_f64.cu so the two halves compile in parallel).
// Whether the segmented kernel takes this shape (16 <= N <= 512, windows free
// of shared-memory bank collisions); otherwise the warp-per-robot kernels.
inline bool sweep_seg_ok(int K, int N, size_t es, bool aligned16) {
    static const bool seg_off = std::getenv("KR_SWEEP_NO_SEG") != nullptr;  // A/B knob
    return !seg_off && N <= 32 * kSegCols && N >= kSegCols &&
           sweep_seg_conflicts(K, N, es, aligned16 && N % 2 == 0) <= 2;
}
// The rotated-window form takes the shapes whose plain windows collide.
inline bool sweep_seg_rot_ok(int K, int N, size_t es, bool aligned16) {
    static const bool rot_off = std::getenv("KR_SWEEP_NO_ROT") != nullptr;  // A/B knob
    return !rot_off && !sweep_seg_ok(K, N, es, aligned16) && N <= 32 * kSegCols && N >= kSegCols &&
           !std::getenv("KR_SWEEP_NO_SEG") &&
           sweep_seg_conflicts(K, N, es, aligned16 && N % 2 == 0, true) <= 2;
}

template <typename T>
int sweep_run(const void* U, int64_t R, int32_t K, int32_t N, int32_t C, int32_t Cc,
              const SweepCfg& cfg, unsigned long long* sums, int32_t* H, uint32_t* flags,
              cudaStream_t st, int max_sms) {
    uint64_t rb = static_cast<uint64_t>(K) * N * sizeof(T);
    const void* bases[1] = {U};
    auto go = [&](auto proto, auto kstaged, auto kdirect) -> int {
        using W = decltype(proto);
        // a warp per robot (32 "items"): 11 consumer warps x 2 robots per tile,
        // two CTAs (24 warps) per SM -- the per-robot scan is instruction-heavy,
        // so warps, not bytes in flight, set the pace
        static const int tr_env = std::getenv("KR_SWEEP_TR") ? std::atoi(std::getenv("KR_SWEEP_TR")) : 0;
        StreamPlan p = make_plan(1, bases, &rb, R, W::kHalf ? 16 : 32, 0, kSweepThreads - 32,
                                 kernel_regs(kstaged), 2,
                                 static_cast<uint32_t>(sizeof(SweepTables)),
                                 tr_env > 0 ? tr_env : (W::kHalf ? 44 : 22));
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
        return launch_stream(kstaged, kdirect, p, w, st, "kr_horizon_sweep", max_sms, cfg);
    };
    // N > 64 (or a misaligned base): a warp per robot, chunks of 32 lanes x VC
    // columns; VC = 2 (pair loads) when the rows allow it.  (VC = 4 was
    // measured 2x slower at N = 128: 0.86 vs 1.75 ms, register spills.)
    const bool al = (reinterpret_cast<uintptr_t>(U) & 15u) == 0;
#define KR_SWEEP(KK, VV) \
    return go(SweepWork<T, KK, VV>{}, k_horizon_sweep<T, KK, VV, true>, k_horizon_sweep<T, KK, VV, false>)
    // segmented sweep: G lanes per robot, <= kSegCols columns per lane
    const bool rot = sweep_seg_rot_ok(K, N, sizeof(T), al);
    if (rot || sweep_seg_ok(K, N, sizeof(T), al)) {
        int G = 1;
        while (G * kSegCols < N) G <<= 1;
        const bool pair = al && N % 2 == 0;
        // pairs: 14-column windows where they cover N (N = 50: 4 x 14)
        const bool c14 = pair && G * 14 >= N;
        const int RW = 32 / G;
        auto go_seg = [&](auto proto, auto kstaged, auto kdirect) -> int {
            using W = decltype(proto);
            static const int tr_env = std::getenv("KR_SWEEP_TR") ? std::atoi(std::getenv("KR_SWEEP_TR")) : 0;
            static const int cw_env = std::getenv("KR_SWEEP_CW") ? std::atoi(std::getenv("KR_SWEEP_CW")) : 0;
            // consumer warps (+ the producer) per CTA, two CTAs per SM: sweeps 5
            // (4 and 5 equal on the common shape, 5 better for fp64 / odd N / ties,
            // 6 leaves one CTA per SM); decide-only launches 4, best beside the
            // round's side stream (profiles/r2_confidence_layouts.jsonl)
            int tr = tr_env > 0 ? tr_env : (cw_env > 0 ? cw_env : (sums ? 5 : 4)) * RW;
            // rotated windows (large robots: N = 64 / 128 / ... fp32): ~36 KB
            // stages -- N = 64: 24 robots, N = 128: 12 (71 -> 91% and 70 -> 90%
            // of the measured peak against 5 warps' worth of robots)
            if (W::kRot && tr_env <= 0 && cw_env <= 0) {
                const int fit = static_cast<int>(36864 / rb) / RW * RW;
                tr = fit > RW ? fit : RW;
            }
            const uint32_t task_bytes = static_cast<uint32_t>((tr * G + 31) / 32) * 32 * kSegCols * 2;
            static const int st_env = std::getenv("KR_SWEEP_STAGES") ? std::atoi(std::getenv("KR_SWEEP_STAGES")) : 0;
            static const int psm_env = std::getenv("KR_SWEEP_PERSM") ? std::atoi(std::getenv("KR_SWEEP_PERSM")) : 0;
            StreamPlan p = make_plan(1, bases, &rb, R, G, 0, kSegThreads - 32, kernel_regs(kstaged), 1,
                                     static_cast<uint32_t>(sizeof(SweepTables)) + task_bytes, tr,
                                     st_env >= 2 ? st_env : kMaxStages);
            p.max_per_sm = psm_env;
            // fp64 keeps the static schedule: the fp64 confidence round's median
            // 494 -> 478 us static (tools/conf_layout_reps.py, 4 interleaved reps)
            p.static_tiles = sizeof(T) == 8;
            if ((R / device_info().sm_count + 1) * static_cast<int64_t>(N) >= (int64_t(1) << 32))
                return KR_EINVAL;
            W w{};
            w.K = K; w.N = N; w.C = C; w.Cc = Cc; w.maxcap = cfg.maxcap; w.half = cfg.half;
            w.G = G; w.RW = RW;
            w.lgRW = 0;
            while ((1 << w.lgRW) < RW) w.lgRW++;
            w.cw = p.threads / 32;
            w.lut_shift = cfg.lut_shift;
            w.lut_base = static_cast<typename W::B>(cfg.clamp_base);
            w.clo = static_cast<T>(cfg.clamp_lo);
            w.chi = static_cast<T>(cfg.clamp_hi);
            w.sfmin = static_cast<T>(cfg.sfmin);
            w.sfmax = static_cast<T>(cfg.sfmax);
            if (cfg.sfmin <= cfg.sfmax) {
                // every element <= emax keeps each (K - 1)-term sum <= sfmax
                const T emax = static_cast<T>(cfg.sfmax / ((K - 1) * 1.01));
                const T smin = static_cast<T>(cfg.sfmin);
                if constexpr (sizeof(T) == 4) {
                    uint32_t a, b;
                    std::memcpy(&a, &emax, 4); std::memcpy(&b, &smin, 4);
                    w.emaxb = a; w.sfminb1 = b - 1;
                } else {
                    uint64_t a, b;
                    std::memcpy(&a, &emax, 8); std::memcpy(&b, &smin, 8);
                    w.emaxb = static_cast<uint32_t>(a >> 32) - 1;  // high word, strictly below
                    w.sfminb1 = b - 1;
                }
            } else {  // no sum filter: every lane re-decides exactly
                w.emaxb = 0;
                w.sfminb1 = ~typename W::B(0);
            }
            w.H = H; w.sums = sums; w.flags = flags; w.R = R;
            // sharing (max_sms > 0): this kernel's CTAs already leave registers and
            // warp slots to the side stream, so every CTA slot of the capped SMs is used
            return launch_stream(kstaged, kdirect, p, w, st, "kr_horizon_sweep",
                                 max_sms > 0 ? -max_sms : max_sms, cfg);
        };
#define KR_SEG(KK, VV, CC)                                                   \
    return go_seg(SweepSeg<T, KK, VV, CC>{}, k_horizon_sweep_seg<T, KK, VV, CC, true>, \
                  k_horizon_sweep_seg<T, KK, VV, CC, false>)
#define KR_SEG_LEAN(KK)                                                                         \
    return go_seg(SweepSeg<T, KK, 2, 14>{}, k_horizon_sweep_seg<T, KK, 2, 14, true, true>,   \
                  k_horizon_sweep_seg<T, KK, 2, 14, false, true>)
#define KR_SEG_ROT(KK, VV)                                                                     \
    return go_seg(SweepSeg<T, KK, VV, 16, true>{}, k_horizon_sweep_seg_rot<T, KK, VV, true>,   \
                  k_horizon_sweep_seg_rot<T, KK, VV, false>)
        if (rot) {
            if (pair) {
                if (K == 6) KR_SEG_ROT(6, 2);
                KR_SEG_ROT(0, 2);
            }
            if (K == 6) KR_SEG_ROT(6, 1);
            KR_SEG_ROT(0, 1);
        }
        if (pair) {
            if (c14) {
                if constexpr (sizeof(T) == 4) {
                    if (!sums) {  // decide-only (confidence horizons): the lean register budget
                        if (K == 6) KR_SEG_LEAN(6);
                        KR_SEG_LEAN(0);
                    }
                }
                if (K == 6) KR_SEG(6, 2, 14);
                KR_SEG(0, 2, 14);
            }
            if (K == 6) KR_SEG(6, 2, 16);
            KR_SEG(0, 2, 16);
        }
        if (K == 6) KR_SEG(6, 1, 16);
        KR_SEG(0, 1, 16);
#undef KR_SEG
#undef KR_SEG_LEAN
#undef KR_SEG_ROT
    }
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
                  cudaStream_t st, int max_sms = 0);
int sweep_run_f64(const void* U, int64_t R, int32_t K, int32_t N, int32_t C, int32_t Cc,
                  const SweepCfg& cfg, unsigned long long* sums, int32_t* H, uint32_t* flags,
                  cudaStream_t st, int max_sms = 0);
int sweep_make_cfg(int dtype, int32_t K, int32_t N, int32_t C, const int32_t* kind,
                   const double* one_plus_t, const int32_t* param, SweepCfg& cfg);

}  // namespace kr
