// kr_sweep.cu -- C entry point of the threshold sweep: configuration table
// (sorted slots, outward-rounded ratio bounds, ratio bucket table) on the host,
// then the per-dtype launcher (kr_sweep_f32.cu / kr_sweep_f64.cu).
#include "kr_sweep.cuh"

using namespace kr;


namespace kr {

// Configuration table of one sweep launch (C <= 64 cells): confidence slots
// first in ascending 1 + t (stable), outward-rounded ratio bounds, the ratio
// bucket table and the segmented kernel's clamp.  KR_EINVAL on a bad cell.
int sweep_make_cfg(int dtype, int32_t K, int32_t N, int32_t C, const int32_t* kind,
                   const double* one_plus_t, const int32_t* param, SweepCfg& cfg) {
    cfg = SweepCfg{};
    // configuration table: confidence slots first, ascending 1 + t (stable)
    int order[kSweepMaxCfg];
    int Cc = 0;
    for (int c = 0; c < C; c++) {
        if (kind[c] != 0 && kind[c] != 1) return KR_EINVAL;
        if (kind[c] == 1) {
            if (!(one_plus_t[c] >= 1.0) || param[c] < 1) return KR_EINVAL;
            order[Cc++] = c;
        } else if (param[c] < 1) {
            return KR_EINVAL;
        }
    }
    for (int a = 1; a < Cc; a++)  // insertion sort (C <= 64)
        for (int b = a; b > 0 && one_plus_t[order[b - 1]] > one_plus_t[order[b]]; b--) {
            const int t = order[b];
            order[b] = order[b - 1];
            order[b - 1] = t;
        }
    int s = Cc;
    for (int c = 0; c < C; c++)
        if (kind[c] == 0) order[s++] = c;
    cfg.C = C;
    cfg.Cc = Cc;
    int P = 1;
    while (P <= Cc) P <<= 1;  // power of two > Cc: table entry P - 1 is +inf
    cfg.half = P / 2;
    // ratio bounds: c = (1 + t) / (K - 1) widened by the filter margin and
    // rounded outward in the storage type
    const bool f32 = dtype == KR_F32;
    const double mrg = f32 ? static_cast<double>(K + 8) * 5.9604644775390625e-8 : 1.7763568394002505e-15;
    for (int i = 0; i < kSweepPad; i++) {
        if (i < Cc) {
            const double c = one_plus_t[order[i]] / static_cast<double>(K - 1);
            if (f32) {
                cfg.rh[i] = std::nextafter(static_cast<float>(c * (1.0 + mrg)), INFINITY);
                cfg.rl[i] = std::nextafter(static_cast<float>(c * (1.0 - mrg)), 0.0f);
            } else {
                cfg.rh[i] = std::nextafter(c * (1.0 + mrg), INFINITY);
                cfg.rl[i] = std::nextafter(c * (1.0 - mrg), 0.0);
            }
        } else {
            cfg.rh[i] = cfg.rl[i] = INFINITY;
        }
    }
    // the filter runs for column sums in [sfmin, sfmax]: every ratio below
    // 2^100 / above 2^-100 of the sum is a normal number in both types
    cfg.sfmin = f32 ? 1e-30 : 1e-290;
    cfg.sfmax = f32 ? 1e30 : 1e290;
    if (!f32 && N < 2) cfg.sfmin = INFINITY;  // fp64 filter assumes the sequential mean order
    // bucket table over [2^floor(log2 rl[0]), 2^(floor(log2 rh[Cc-1]) + 1)):
    // 2^mbits buckets per binade
    cfg.lut_n = 1;  // default: one ambiguous bucket covering everything
    cfg.lut_lo = 0;
    cfg.lut_hi = f32 ? 0xFFFFFFFFull : ~uint64_t(0);  // above the largest ratio pattern
    cfg.lut_shift = f32 ? 31 : 63;
    cfg.lut[0] = 0xFFFF;
    bool table = false;
    if (Cc > 0 && std::isnormal(cfg.rl[0]) && std::isfinite(cfg.rh[Cc - 1]) &&
        (!f32 || (cfg.rl[0] > 1e-37 && cfg.rh[Cc - 1] < 1e37))) {
        int e_lo, e_hi;
        std::frexp(cfg.rl[0], &e_lo);       // rl[0] in [2^(e_lo-1), 2^e_lo)
        std::frexp(cfg.rh[Cc - 1], &e_hi);  // rh    in [2^(e_hi-1), 2^e_hi)
        const double lo = std::ldexp(1.0, e_lo - 1), hi = std::ldexp(1.0, e_hi);
        const int binades = e_hi - e_lo + 1;
        int mbits = 7;
        while (mbits > 0 && (binades << mbits) > kSweepLut) mbits--;
        if ((binades << mbits) <= kSweepLut && (f32 || binades < 2000)) {
            const int mant = f32 ? 23 : 52;
            cfg.lut_shift = mant - mbits;
            cfg.lut_n = binades << mbits;
            auto bits_of = [&](double x) -> uint64_t {
                if (f32) { const float f = static_cast<float>(x); uint32_t b; std::memcpy(&b, &f, 4); return b; }
                uint64_t b; std::memcpy(&b, &x, 8); return b;
            };
            auto val_of = [&](uint64_t b) -> double {
                if (f32) { const uint32_t b32 = static_cast<uint32_t>(b); float f; std::memcpy(&f, &b32, 4); return f; }
                double d; std::memcpy(&d, &b, 8); return d;
            };
            cfg.lut_lo = bits_of(lo);
            cfg.lut_hi = bits_of(hi);
            table = true;
            // both counts are monotone in the bucket (rh, rl ascending): two pointers
            int a = 0, nb = 0;
            for (int bkt = 0; bkt < cfg.lut_n; bkt++) {
                const uint64_t b0 = cfg.lut_lo + (static_cast<uint64_t>(bkt) << cfg.lut_shift);
                const double x0 = val_of(b0);
                const double x1 = val_of(b0 + (uint64_t(1) << cfg.lut_shift) - 1);  // largest in bucket
                while (a < Cc && cfg.rh[a] < x0) a++;    // every ratio in the bucket is a definite trip
                while (nb < Cc && cfg.rl[nb] <= x1) nb++;  // some ratio is not a definite non-trip
                cfg.lut[bkt] = a == nb ? static_cast<uint16_t>(a) : uint16_t(0xFFFF);
            }
        }
    }
    // segmented kernel: the ratio is clamped to [clamp_lo, clamp_hi] so that
    // (bits(ratio) - clamp_base) >> lut_shift indexes [below, table, above]
    if (table) {
        const uint64_t step = uint64_t(1) << cfg.lut_shift;
        cfg.clamp_base = cfg.lut_lo - step;
        if (f32) {
            const uint32_t lo32 = static_cast<uint32_t>(cfg.clamp_base), hi32 = static_cast<uint32_t>(cfg.lut_hi);
            float a, b;
            std::memcpy(&a, &lo32, 4); std::memcpy(&b, &hi32, 4);
            cfg.clamp_lo = a; cfg.clamp_hi = b;
        } else {
            std::memcpy(&cfg.clamp_lo, &cfg.clamp_base, 8);
            std::memcpy(&cfg.clamp_hi, &cfg.lut_hi, 8);
        }
        cfg.lut_below = 0;
        cfg.lut_above = static_cast<uint16_t>(Cc);
    } else {  // no table: every ratio lands on an undecided entry
        cfg.clamp_base = 0;
        cfg.clamp_lo = 0.0;
        cfg.clamp_hi = INFINITY;
        cfg.lut_below = cfg.lut_above = 0xFFFF;
    }
    for (int i = 0; i < C; i++) {
        const int c = order[i];
        cfg.orig[i] = c;
        cfg.hcap[i] = param[c] < N ? param[c] : N;  // horizon.py:121-122, 130-131
        if (i < Cc) {
            cfg.p[i] = one_plus_t[c];
            if (cfg.hcap[i] > cfg.maxcap) cfg.maxcap = cfg.hcap[i];
        }
    }
    return KR_OK;
}

}  // namespace kr

extern "C" int kr_horizon_sweep(const void* U, int dtype, int64_t R, int32_t K, int32_t N,
                                int32_t C, const int32_t* kind, const double* one_plus_t,
                                const int32_t* param, unsigned long long* sums, int32_t* H,
                                uint32_t* flags, void* stream) {
    if (R < 0 || K < 2 || N < 1 || C < 1 || C > kSweepMaxCfg || !kind || !one_plus_t || !param ||
        (dtype != KR_F32 && dtype != KR_F64))
        return KR_EINVAL;
    if (R == 0) return KR_OK;
    if (!U || !sums) return KR_EINVAL;
    if (N > (kStreamThreads - 32) * kMaxRounds) return KR_EINVAL;
    SweepCfg cfg;
    const int rc = sweep_make_cfg(dtype, K, N, C, kind, one_plus_t, param, cfg);
    if (rc != KR_OK) return rc;
    const int Cc = cfg.Cc;
    cudaStream_t st = as_stream(stream);
    return dtype == KR_F64 ? sweep_run_f64(U, R, K, N, C, Cc, cfg, sums, H, flags, st)
                           : sweep_run_f32(U, R, K, N, C, Cc, cfg, sums, H, flags, st);
}
