// kr_select_state.cuh -- the radix select's device state, shared by the
// select kernels (kr_select.cu) and the planning round's urgency pass, whose
// last CTA prepares the state for the select (kr_urgency_prep), so the round's
// side stream needs no state-reset or statistics-init launches.
#pragma once
#include "kr_common.cuh"

namespace kr {

constexpr int kDigitBits = 11;
constexpr int kBins = 1 << kDigitBits;

// Digit = the values of the candidate set's kDigitBits most significant
// *differing* bit positions (a pext of OR ^ AND), MSB first.  All candidates
// agree on every other bit, so digit order is key order; unlike a contiguous
// bit window it never wastes digit bits on constant fields (e.g. the high
// zero bits of the aged estimate between the bucket and its significant bits).
struct Digit {
    int W;                 // number of digit bits (0: all candidates identical)
    int nrun;              // the digit bits grouped into runs of adjacent positions
    int run_pos[kDigitBits];  // lowest bit position (0..127) of each run, MSB run first
    int run_len[kDigitBits];
    bool any;
};
struct SelState {
    unsigned long long st[2][4];  // [parity] {or_hi, or_lo, and_hi, and_lo}
    unsigned int cnt[2];          // [parity] candidate count
    long long need;               // 1-based rank of the target within candidates
    unsigned int dstar;
    unsigned int dcount;          // population of the boundary bin
    int done;
    int pad_;
    kr_key kth;
    unsigned int sel_count;       // admission gather count
    unsigned int pad2_[3];
    unsigned long long sst[4];    // OR/AND of the gathered (admitted) keys
    Digit d0;                     // level-0 digit (from the keys' OR / AND)
    unsigned int dstar0;          // its boundary bin (dstar moves on in later levels)
    unsigned int done_hist;       // last-CTA-done counters of the two grid passes
    unsigned int done_scatter;
    unsigned int done_urg;        // last-CTA counter of the preparing urgency pass
    unsigned int hist[kBins];
};

// Built with compile-time indices only (predicated updates) so that the run
// table lives in registers for the per-key extraction loops.
__device__ __forceinline__ Digit digit_of(const unsigned long long* s) {
    unsigned long long xlo = s[1] ^ s[3], xhi = s[0] ^ s[2];
    Digit d;
    d.W = 0;
    d.nrun = 0;
#pragma unroll
    for (int r = 0; r < kDigitBits; r++) {
        d.run_pos[r] = 0;
        d.run_len[r] = 0;
    }
    int last = -2;
#pragma unroll
    for (int w = 0; w < kDigitBits; w++) {
        int pos = -1;
        if (xhi) {
            pos = 127 - __clzll(xhi);
            xhi &= ~(1ull << (pos - 64));
        } else if (xlo) {
            pos = 63 - __clzll(xlo);
            xlo &= ~(1ull << pos);
        }
        if (pos >= 0) {
            // extend the current run downwards unless it would cross the word boundary
            const bool extend = pos == last - 1 && (pos >> 6) == (last >> 6);
            const int cur = extend ? d.nrun - 1 : d.nrun;
#pragma unroll
            for (int r = 0; r < kDigitBits; r++) {
                if (r == cur) {
                    d.run_pos[r] = pos;
                    d.run_len[r] += 1;
                }
            }
            d.nrun = cur + 1;
            last = pos;
            d.W = w + 1;
        }
    }
    d.any = d.W > 0;
    return d;
}

__device__ __forceinline__ void sel_init(SelState* s, int64_t n, int64_t k) {
    s->st[1][0] = 0; s->st[1][1] = 0; s->st[1][2] = ~0ull; s->st[1][3] = ~0ull;
    s->sst[0] = 0; s->sst[1] = 0; s->sst[2] = ~0ull; s->sst[3] = ~0ull;
    s->cnt[0] = static_cast<unsigned>(n);
    s->cnt[1] = 0;
    s->need = k;
    s->done = 0;
    s->sel_count = 0;
    s->done_hist = 0;
    s->done_scatter = 0;
}
// The level-0 digit of the full key set; a set of identical keys (n == 1,
// keys being unique) is its own answer.
__device__ __forceinline__ void sel_digit0(SelState* s, const kr_key* keys) {
    s->d0 = digit_of(s->st[0]);
    if (!s->d0.any) {
        s->kth = keys[0];
        s->done = 1;
    }
}

// The select state for a round over n keys with budget k, from the keys'
// OR / AND statistics st4 {or_hi, or_lo, and_hi, and_lo}.  Run by every thread
// of one CTA after all keys are written (the urgency pass's last CTA).
__device__ __forceinline__ void sel_prepare(SelState* s, int64_t n, int64_t k,
                                            const unsigned long long* st4, const kr_key* keys) {
    for (int i = threadIdx.x; i < kBins; i += blockDim.x) s->hist[i] = 0;
    if (threadIdx.x == 0) {
        for (int j = 0; j < 4; j++) s->st[0][j] = st4[j];
        sel_init(s, n, k);
        sel_digit0(s, keys);
        s->done_urg = 0;
    }
}

}  // namespace kr
