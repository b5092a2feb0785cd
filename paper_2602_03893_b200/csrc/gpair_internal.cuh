// gpair_internal.cuh -- shared device helpers of the B200 GPAIR hot path.
//
// Per-pair arithmetic of Eq. 7 with the 3-sigma window
// of P:291, in SAMPLE UNITS (u = d / h, h = v / f_s), so that stepping from
// one sample to the next (u - m) is exact in fp32:
//
//   value(n) = A d exp(-d^2/2 sigma^2) / (2 r) = w' u exp2(K1u u^2),
//   w' = A h / (2 r),  K1u = -log2(e) h^2 / (2 sigma^2),  u = (r - v t_n) / h.
//
// Two-level time of flight:
//   * fp64 anchor per (8-kernel group g, sensor j): R = |C_g - s_j|,
//     n_a = floor((R/v - t0) f_s), Eu = (R - v t_{n_a}) / h   (u at sample n_a)
//   * fp32 per-pair offset from q = 2 (C_g - s_j).delta + |delta|^2,
//     delta = c_i - C_g:  (r - R)/h = (q / (2 R h)) S(eps),  eps = q / R^2,
//     S = 1 - eps/4 + eps^2/8 - 5 eps^3/64 + 7 eps^4/128 - 21 eps^5/512
//     (series of (sqrt(1+eps)-1)/(eps/2)), and h/(2r) = (h/(2R)) T(eps),
//     T = 1 - eps/2 + 3eps^2/8 - 5eps^3/16 + 35eps^4/128 (series of (1+eps)^-1/2).
//     Groups whose eps could exceed EPS_FAST use an exact per-pair fp64 path.
//   * window membership |d| < k sigma decided in fp32 unless an edge is
//     within GAMMA samples of a sample point; then the pair is re-decided
//     bit-identically to the fp64 oracle (same operations, IEEE fp64).
//   * one MUFU ex2 per in-window sample (SFU), accumulated in fp32.
// See DESIGN.md "Numerics" for the error budget of each step.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace gpair {

constexpr int CELL = 32;          // kernels per cell (one warp lane each in the adjoint)
constexpr int GROUP = 8;          // kernels per fp64 anchor (2x2x2 on a grid)
constexpr int GPC = CELL / GROUP; // groups per cell
constexpr float GAMMA = 4e-5f;    // ambiguity band of the fp32 window edges [samples]
constexpr double EPS_FAST = 0.03; // max |eps| of the series path (else exact fp64 per pair)
constexpr double MAX_DR_SAMPLES = 4.0; // max group radius [samples] of the series path
constexpr double EPS_SMALL = 0.006;    // max |eps| for the degree-2 series (SER = 2)
constexpr float RND_MAGIC = 12582912.f;      // 1.5 * 2^23
constexpr int RND_MAGIC_BITS = 0x4B400000;   // __float_as_int(RND_MAGIC)
#ifndef GPAIR_ADJ_ACC64
#define GPAIR_ADJ_ACC64 1
#endif
// Accumulator of the sensor-lane adjoints' cross-sensor sums (warp reduce-scatter,
// per-warp smem sums, sensor-group partials, k_adj_gather): fp64 keeps these
// sums' rounding out of the gradient's error budget.
#if GPAIR_ADJ_ACC64
typedef double gacc_t;
#else
typedef float gacc_t;
#endif

// Operator constants, computed once on the host in fp64 and passed by value.
struct OpConst {
    double v, fs, t0, ks;  // ks = k * sigma (fp64, same bits as the oracle's k*sigma)
    double h;              // v / f_s [m]
    double inv_h;          // f_s / v
    double t0fs;           // t0 * f_s
    int32_t Nt, Nd;
    int32_t wmax;          // max in-window count of any pair
    int32_t cnt_int;       // 2 k sigma / h if it is an integer (fp32 ku exact), else 0
    float c_lo;            // -ku - 1/2   (pair_fast)
    float c_u;             // ku - 1/2    (pair_fast)
    float ku;              // k sigma / h  [samples]
    float K1u;             // -log2(e) h^2 / (2 sigma^2)
    // ASSA operator (row f1, Eqs. 8-12); alpha = 0 for the exact operator
    int32_t alpha;         // upsampling ratio
    int32_t K;             // taps half-width alpha N_half
    int32_t n_half;        // N_half
    double fs_up;          // alpha f_s (computed as (double)alpha * fs, like the oracle)
    float two_over_h;      // 2 / h: (A h / 2r) * (2/h) = A / r
    double win_half;       // half-width [m] of the conservative sample windows (setup)
    // general operator (row f4): per-kernel sigma_i and/or the near-field term
    double kwin;           // window k (fp64, the oracle's k in k * sigma_i)
    int32_t gen;           // 1: per-kernel sigma table / near-field (kernel path SER_GEN)
    int32_t nf;            // 1: near-field operator (Eq. 6, both terms; reading N1)
    double nf_add;         // max(0, -v t0): near pairs are r < k sigma_i + nf_add (+ margin)
    double nf_thr_max;     // bound of every pair's near threshold; -1 when nf = 0
    int32_t per_sigma;     // 1: sigma_i from the table (desc.sigmas); 0: the scalar sigma
    double sigma;          // scalar sigma (fp64, as given)
    // launch-local offsets of the sensor-group pipeline (gpair_api.cu iterate_pipelined):
    // forward / sensor-lane adjoint CTAs use sensor group blockIdx.y + grp0, reducer CTAs sensor blockIdx.x + j0
    int32_t grp0;
    int32_t j0;
};

constexpr int SER_GEN = 7;    // kernel path of the general operator (pair_gen)
constexpr int SER_FAST5 = 6;  // fast packed path (exact-integer window) with the degree-5 series (|eps| <= EPS_FAST)

// Near-pair threshold of reading N1: pairs with r < thr are evaluated with
// both terms of Eq. 6 by gpair_near.cu; the rest carry only the outgoing
// term (their incoming window is empty; the relative margin only moves a few
// more pairs to the exact near path).  Used identically by the near-list
// builder and the main kernels' exact path.
__device__ __forceinline__ double kernel_sigma(float sigma_i, const OpConst& k) {
    return k.per_sigma ? (double)sigma_i : k.sigma;
}
// k sigma_i exactly as the oracle forms it (`double ks = k * s;`)
__device__ __forceinline__ double kernel_ks(float sigma_i, const OpConst& k) {
    return k.per_sigma ? __dmul_rn(k.kwin, (double)sigma_i) : k.ks;
}
__device__ __forceinline__ double near_threshold(double ks, const OpConst& k) {
    return __dadd_rn(__dmul_rn(__dadd_rn(ks, k.nf_add), 1.0 + 1e-9), 1e-15);
}

// fp64 anchor of a (group, sensor) pair, reduced to what the per-pair fp32
// arithmetic needs.  na == NA_EXACT: use the per-pair fp64 path.
struct __align__(16) Anchor {
    float Ux, Uy, Uz;  // 2 (C_g - s_j)
    float Eu;          // (R - v t_{n_a}) / h, in [0, 1) up to rounding
    float invR2;       // 1 / R^2
    float inv2Rh;      // 1 / (2 R h)
    float h2R;         // h / (2 R)
    int32_t na;        // anchor sample index floor((R/v - t0) f_s)
};

constexpr int32_t NA_EXACT = -2147483647 - 1;

__device__ __forceinline__ Anchor make_anchor(float4 C, float sx, float sy, float sz, const OpConst& k,
                                              double* invR_out = nullptr) {
    const double dx = (double)C.x - (double)sx;
    const double dy = (double)C.y - (double)sy;
    const double dz = (double)C.z - (double)sz;
    const double R2 = fma(dx, dx, fma(dy, dy, dz * dz));
    const double invR = rsqrt(R2);
    const double R = R2 * invR;
    if (invR_out) *invR_out = invR;
    const double tf = fma(R, k.inv_h, -k.t0fs);  // (R/v - t0) f_s in samples
    const double na = floor(tf);
    Anchor a;
    a.Ux = (float)(2.0 * dx);
    a.Uy = (float)(2.0 * dy);
    a.Uz = (float)(2.0 * dz);
    a.Eu = (float)(tf - na);  // exact fp64 subtraction
    a.invR2 = (float)(invR * invR);
    a.inv2Rh = (float)(0.5 * invR * k.inv_h);
    a.h2R = (float)(0.5 * k.h * invR);
    // series accuracy: |eps| <= (2 R rad + rad^2) / R^2 (C.w = group radius)
    const double rad = C.w;
    const bool series_ok = fma(2.0 * R, rad, rad * rad) <= EPS_FAST * R2 && rad <= MAX_DR_SAMPLES * k.h &&
                           R - rad > k.nf_thr_max;  // near pairs (row f4) always take the exact path
    a.na = series_ok ? (int32_t)na : NA_EXACT;
    return a;
}

// Exact (oracle-identical) window of one pair: first and last n with
// |r - v (t0 + n/f_s)| < ks, clipped to [0, N_t).  d(n) = r - v t_n is
// monotone in n (every rounding step is monotone), so the window is found by
// walking from the fp32 guesses g_first / g_last (accurate to +-1 sample).
// r comes from the ORIGINAL fp32 inputs in fp64 with explicit
// round-to-nearest ops (no FMA contraction), exactly like the oracle's
// pair_distance() and membership test, so the decision is bit-identical.
__device__ __forceinline__ double exact_r(float cx, float cy, float cz, float sx, float sy, float sz) {
    double dx = __dsub_rn((double)cx, (double)sx);
    double dy = __dsub_rn((double)cy, (double)sy);
    double dz = __dsub_rn((double)cz, (double)sz);
    double r2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
    return __dsqrt_rn(r2);
}

__device__ __forceinline__ double exact_d(double r, int n, const OpConst& k) {
    double t = __dadd_rn(k.t0, __ddiv_rn((double)n, k.fs));
    return __dsub_rn(r, __dmul_rn(k.v, t));
}

__device__ __forceinline__ void exact_window(double r, int g_first, int g_last, const OpConst& k,
                                                 int& n_lo, int& cnt, double ks) {
    int f = g_first;
    while (exact_d(r, f - 1, k) < ks) --f;
    while (!(exact_d(r, f, k) < ks)) ++f;
    int l = g_last;
    while (exact_d(r, l + 1, k) > -ks) ++l;
    while (!(exact_d(r, l, k) > -ks)) --l;
    if (f < 0) f = 0;
    if (l > k.Nt - 1) l = k.Nt - 1;
    n_lo = f;
    cnt = l - f + 1;
    if (cnt < 0) cnt = 0;
}

// Exact per-pair fp64 time of flight for groups outside the series' range.
__device__ __forceinline__ void exact_pair(float cx, float cy, float cz, float sx, float sy, float sz,
                                               float A, const OpConst& k, float& eu, float& w, int& na,
                                               double& r) {
    r = exact_r(cx, cy, cz, sx, sy, sz);
    double nad = floor((r / k.v - k.t0) * k.fs);
    eu = (float)((r - k.v * (k.t0 + nad / k.fs)) / k.h);
    w = (float)((double)A * 0.5 * k.h / r);
    na = (int)nad;
}

struct PairWin {
    float u_lo;   // u = d / h at the first in-window sample
    float w;      // A h / (2 r)
    int32_t n_lo; // first in-window sample
    int32_t cnt;  // number of in-window samples (0 = none)
};

// Per-pair window and weight.  kd = (dx, dy, dz, |d|^2) relative to the group
// anchor; orig = original centres, read only on the rare exact paths.
// SER = 5: series to eps^5 / eps^4 (|eps| <= EPS_FAST); SER = 2: to eps^2
// (|eps| <= EPS_SMALL, truncation <= 7e-8 relative; chosen at create).
template <int SER>
__device__ __forceinline__ PairWin pair_setup(const Anchor& a, float4 kd, float A, const float* __restrict__ orig,
                                              int64_t gi, int64_t Mpad, float sx, float sy, float sz,
                                              const OpConst& k) {
    PairWin p;
    float eu;
    int na;
    if (a.na != NA_EXACT) {
        const float q = fmaf(a.Ux, kd.x, fmaf(a.Uy, kd.y, fmaf(a.Uz, kd.z, kd.w)));
        const float eps = q * a.invR2;
        float S, Tw;
        if (SER == 2) {
            S = fmaf(eps, fmaf(eps, 1.f / 8.f, -0.25f), 1.f);
            Tw = fmaf(eps, fmaf(eps, 3.f / 8.f, -0.5f), 1.f);
        } else {
            S = fmaf(eps, -21.f / 512.f, 7.f / 128.f);
            S = fmaf(eps, S, -5.f / 64.f);
            S = fmaf(eps, S, 1.f / 8.f);
            S = fmaf(eps, S, -0.25f);
            S = fmaf(eps, S, 1.f);
            Tw = fmaf(eps, 35.f / 128.f, -5.f / 16.f);
            Tw = fmaf(eps, Tw, 3.f / 8.f);
            Tw = fmaf(eps, Tw, -0.5f);
            Tw = fmaf(eps, Tw, 1.f);
        }
        eu = fmaf(q * a.inv2Rh, S, a.Eu);  // u at sample n_a
        p.w = A * (a.h2R * Tw);
        na = a.na;
    } else {
        double r_ex;
        exact_pair(orig[gi], orig[Mpad + gi], orig[2 * Mpad + gi], sx, sy, sz, A, k, eu, p.w, na, r_ex);
    }
    // In-window m satisfy alpha < m < beta (alpha = eu - ku, beta = eu + ku).
    // floor() without the XU pipe: for |x| < 2^22, (x + 1.5*2^23) rounds x to
    // the nearest integer, held in the low mantissa bits.  floor(alpha) =
    // rint(alpha - 1/2) whenever alpha is not within GAMMA of an integer; the
    // ambiguous case goes to the exact path anyway.
    const float alpha = eu - k.ku;
    const float ta = (alpha - 0.5f) + RND_MAGIC;
    const float fla = ta - RND_MAGIC;
    bool amb = fabsf((alpha - fla) - 0.5f) > 0.5f - GAMMA;
    int n_lo = na + (__float_as_int(ta) - RND_MAGIC_BITS) + 1;
    int n_hi;
    float u_lo = eu - (fla + 1.f);  // exact: integer shift of a small float
    if (k.cnt_int > 0) {
        // 2 ku is an exact integer: frac(beta) = frac(alpha), so the window
        // holds exactly cnt_int samples unless alpha is ambiguous
        n_hi = n_lo + k.cnt_int - 1;
    } else {
        const float beta = eu + k.ku;
        const float tb = (beta - 0.5f) + RND_MAGIC;
        amb = amb || fabsf((beta - (tb - RND_MAGIC)) - 0.5f) > 0.5f - GAMMA;
        n_hi = na + (__float_as_int(tb) - RND_MAGIC_BITS);  // ceil(beta) - 1 = floor(beta)
    }
    if (amb || n_lo < 0 || n_hi > k.Nt - 1) {  // rare: exact edges and/or record clipping
        if (amb) {
            const double r = exact_r(orig[gi], orig[Mpad + gi], orig[2 * Mpad + gi], sx, sy, sz);
            int cnt;
            exact_window(r, n_lo, n_hi, k, n_lo, cnt, k.ks);
            n_hi = n_lo + cnt - 1;
        } else {
            n_lo = max(n_lo, 0);
            n_hi = min(n_hi, k.Nt - 1);
        }
        u_lo = eu - (float)(n_lo - na);
    }
    p.n_lo = n_lo;
    p.cnt = max(n_hi - n_lo + 1, 0);
    p.u_lo = u_lo;
    return p;
}

// Rare path of pair_fast(): exact window edges and/or record clipping.
static __device__ __noinline__ PairWin pair_fix(PairWin p, float eu, int na, bool amb, const float* __restrict__ orig,
                                                int64_t gi, int64_t Mpad, float sx, float sy, float sz, int cnt_guess,
                                                const OpConst k) {
    int n_lo = p.n_lo, n_hi = p.n_lo + cnt_guess - 1;
    if (amb) {
        const double r = exact_r(orig[gi], orig[Mpad + gi], orig[2 * Mpad + gi], sx, sy, sz);
        int cnt;
        exact_window(r, n_lo, n_hi, k, n_lo, cnt, k.ks);
        n_hi = n_lo + cnt - 1;
    } else {
        n_lo = max(n_lo, 0);
        n_hi = min(n_hi, k.Nt - 1);
    }
    p.n_lo = n_lo;
    p.cnt = max(n_hi - n_lo + 1, 0);
    p.u_lo = eu - (float)(n_lo - na);
    return p;
}

// Fast per-pair setup for the common configuration (FAST): degree-2 series
// (every |eps| <= EPS_SMALL), window length 2 k sigma / h an exact integer
// (k.cnt_int), anchor not exact.  Same arithmetic as pair_setup<2> with the
// constants folded: x = eu - ku - 1/2, fl = rint(x) = floor(alpha),
// u_lo = eu - (fl + 1).
__device__ __forceinline__ PairWin pair_fast(const Anchor& a, float4 kd, float A, const float* __restrict__ orig,
                                             int64_t gi, int64_t Mpad, float sx, float sy, float sz,
                                             const OpConst& k) {
    PairWin p;
    const float q = fmaf(a.Ux, kd.x, fmaf(a.Uy, kd.y, fmaf(a.Uz, kd.z, kd.w)));
    const float eps = q * a.invR2;
    const float S = fmaf(eps, fmaf(eps, 1.f / 8.f, -0.25f), 1.f);
    const float Tw = fmaf(eps, fmaf(eps, 3.f / 8.f, -0.5f), 1.f);
    const float eu = fmaf(q * a.inv2Rh, S, a.Eu);
    p.w = A * (a.h2R * Tw);
    const float x = eu + k.c_lo;              // alpha - 1/2
    const float t = x + RND_MAGIC;
    const float fl = t - RND_MAGIC;           // floor(alpha) unless ambiguous
    const float d = x - fl;                   // frac(alpha) - 1/2
    p.n_lo = a.na + __float_as_int(t) - (RND_MAGIC_BITS - 1);
    p.u_lo = eu - (fl + 1.f);                 // u at n_lo (exact: no rounding of x leaks in)
    p.cnt = k.cnt_int;
    const bool amb = fabsf(d) > 0.5f - GAMMA;
    if (amb || (unsigned)p.n_lo > (unsigned)(k.Nt - k.cnt_int))
        p = pair_fix(p, eu, a.na, amb, orig, gi, Mpad, sx, sy, sz, k.cnt_int, k);
    return p;
}

// General per-pair setup (row f4; kernel path SER_GEN): per-kernel sigma_i
// from ks4 = (k sigma_i / h, -log2(e) h^2 / (2 sigma_i^2), sigma_i, 0) and,
// when k.nf, near pairs (r < near_threshold) skipped here: gpair_near.cu
// evaluates them with both terms of Eq. 6.  Same window logic as
// pair_setup<5> with the per-kernel half-width; ambiguous edges are decided
// in fp64 against k sigma_i computed like the oracle's `k * s`.
__device__ __forceinline__ PairWin pair_gen(const Anchor& a, float4 kd, float A, float4 ks4,
                                            const float* __restrict__ orig, int64_t gi, int64_t Mpad, float sx,
                                            float sy, float sz, const OpConst& k) {
    PairWin p;
    float eu;
    int na;
    double r = -1.0;
    if (a.na != NA_EXACT) {
        const float q = fmaf(a.Ux, kd.x, fmaf(a.Uy, kd.y, fmaf(a.Uz, kd.z, kd.w)));
        const float eps = q * a.invR2;
        float S = fmaf(eps, -21.f / 512.f, 7.f / 128.f);
        S = fmaf(eps, S, -5.f / 64.f);
        S = fmaf(eps, S, 1.f / 8.f);
        S = fmaf(eps, S, -0.25f);
        S = fmaf(eps, S, 1.f);
        float Tw = fmaf(eps, 35.f / 128.f, -5.f / 16.f);
        Tw = fmaf(eps, Tw, 3.f / 8.f);
        Tw = fmaf(eps, Tw, -0.5f);
        Tw = fmaf(eps, Tw, 1.f);
        eu = fmaf(q * a.inv2Rh, S, a.Eu);
        p.w = A * (a.h2R * Tw);
        na = a.na;
    } else {
        exact_pair(orig[gi], orig[Mpad + gi], orig[2 * Mpad + gi], sx, sy, sz, A, k, eu, p.w, na, r);
        if (k.nf && r < near_threshold(kernel_ks(ks4.z, k), k)) {
            p.cnt = 0;
            p.n_lo = 0;
            p.u_lo = 0.f;
            return p;
        }
    }
    const float alpha = eu - ks4.x;
    const float ta = (alpha - 0.5f) + RND_MAGIC;
    const float fla = ta - RND_MAGIC;
    bool amb = fabsf((alpha - fla) - 0.5f) > 0.5f - GAMMA;
    int n_lo = na + (__float_as_int(ta) - RND_MAGIC_BITS) + 1;
    const float beta = eu + ks4.x;
    const float tb = (beta - 0.5f) + RND_MAGIC;
    amb = amb || fabsf((beta - (tb - RND_MAGIC)) - 0.5f) > 0.5f - GAMMA;
    int n_hi = na + (__float_as_int(tb) - RND_MAGIC_BITS);
    float u_lo = eu - (fla + 1.f);
    if (amb || n_lo < 0 || n_hi > k.Nt - 1) {
        if (amb) {
            if (r < 0.0) r = exact_r(orig[gi], orig[Mpad + gi], orig[2 * Mpad + gi], sx, sy, sz);
            int cnt;
            exact_window(r, n_lo, n_hi, k, n_lo, cnt, kernel_ks(ks4.z, k));
            n_hi = n_lo + cnt - 1;
        } else {
            n_lo = max(n_lo, 0);
            n_hi = min(n_hi, k.Nt - 1);
        }
        u_lo = eu - (float)(n_lo - na);
    }
    p.n_lo = n_lo;
    p.cnt = max(n_hi - n_lo + 1, 0);
    p.u_lo = u_lo;
    return p;
}

// ---- ASSA (row f1): aligned upsampled index k_ij and weight A / r_ij.
// k_ij = floor((r/v - t0) f_s^up + 0.5) = alpha n_a + floor(alpha eu + 1/2)
// (alpha n_a is an exact integer).  When alpha eu + 1/2 is within
// GAMMA * alpha of an integer the index is re-decided in fp64 with the
// oracle's exact operations (gpair_oracle.c assa_index()).
struct AssaPair {
    int32_t k;   // aligned index on the upsampled grid (may be outside [0, alpha N_t))
    float w;     // A / r
};

__device__ __forceinline__ int64_t assa_exact_k(double r, const OpConst& k) {
    double q = __ddiv_rn(r, k.v);
    q = __dsub_rn(q, k.t0);
    q = __dmul_rn(q, k.fs_up);
    q = __dadd_rn(q, 0.5);
    return (int64_t)floor(q);
}

template <int SER>
__device__ __forceinline__ AssaPair assa_setup(const Anchor& a, float4 kd, float A, const float* __restrict__ orig,
                                               int64_t gi, int64_t Mpad, float sx, float sy, float sz,
                                               const OpConst& k) {
    AssaPair p;
    float eu, w;
    int na;
    if (a.na != NA_EXACT) {
        const float q = fmaf(a.Ux, kd.x, fmaf(a.Uy, kd.y, fmaf(a.Uz, kd.z, kd.w)));
        const float eps = q * a.invR2;
        float S, Tw;
        if (SER <= 2) {
            S = fmaf(eps, fmaf(eps, 1.f / 8.f, -0.25f), 1.f);
            Tw = fmaf(eps, fmaf(eps, 3.f / 8.f, -0.5f), 1.f);
        } else {
            S = fmaf(eps, -21.f / 512.f, 7.f / 128.f);
            S = fmaf(eps, S, -5.f / 64.f);
            S = fmaf(eps, S, 1.f / 8.f);
            S = fmaf(eps, S, -0.25f);
            S = fmaf(eps, S, 1.f);
            Tw = fmaf(eps, 35.f / 128.f, -5.f / 16.f);
            Tw = fmaf(eps, Tw, 3.f / 8.f);
            Tw = fmaf(eps, Tw, -0.5f);
            Tw = fmaf(eps, Tw, 1.f);
        }
        eu = fmaf(q * a.inv2Rh, S, a.Eu);
        w = A * (a.h2R * Tw);
        na = a.na;
    } else {
        double r_ex;
        exact_pair(orig[gi], orig[Mpad + gi], orig[2 * Mpad + gi], sx, sy, sz, A, k, eu, w, na, r_ex);
    }
    p.w = w * k.two_over_h;
    const float xa = fmaf((float)k.alpha, eu, 0.5f);
    const float t = (xa - 0.5f) + RND_MAGIC;  // rint(xa - 1/2) = floor(xa) unless ambiguous
    const float fl = t - RND_MAGIC;
    const bool amb = fabsf((xa - fl) - 0.5f) > 0.5f - GAMMA * (float)k.alpha;
    if (amb) {
        const double r = exact_r(orig[gi], orig[Mpad + gi], orig[2 * Mpad + gi], sx, sy, sz);
        p.k = (int32_t)assa_exact_k(r, k);
    } else {
        p.k = k.alpha * na + (__float_as_int(t) - RND_MAGIC_BITS);
    }
    return p;
}

// Rare path of assa_fast(): exact fp64 re-decision of k_ij.
static __device__ __noinline__ int assa_fix(const float* __restrict__ orig, int64_t gi, int64_t Mpad, float sx,
                                            float sy, float sz, const OpConst k) {
    const double r = exact_r(orig[gi], orig[Mpad + gi], orig[2 * Mpad + gi], sx, sy, sz);
    return (int)assa_exact_k(r, k);
}

// Branch-free part of assa_fast(): k guess, weight and the ambiguity flag, so
// that several pairs can be set up back to back (instruction-level parallelism)
// before one shared rare-path branch.
struct AssaPre {
    int32_t k;
    float w;
    bool amb;
};
__device__ __forceinline__ AssaPre assa_pre(const Anchor& a, float4 kd, float A, const OpConst& k) {
    AssaPre p;
    const float q = fmaf(a.Ux, kd.x, fmaf(a.Uy, kd.y, fmaf(a.Uz, kd.z, kd.w)));
    const float eps = q * a.invR2;
    const float S = fmaf(eps, fmaf(eps, 1.f / 8.f, -0.25f), 1.f);
    const float Tw = fmaf(eps, fmaf(eps, 3.f / 8.f, -0.5f), 1.f);
    const float eu = fmaf(q * a.inv2Rh, S, a.Eu);
    p.w = (A * (a.h2R * Tw)) * k.two_over_h;
    const float xa = fmaf((float)k.alpha, eu, 0.5f);
    const float t = (xa - 0.5f) + RND_MAGIC;
    const float fl = t - RND_MAGIC;
    p.k = k.alpha * a.na + (__float_as_int(t) - RND_MAGIC_BITS);
    p.amb = fabsf((xa - fl) - 0.5f) > 0.5f - GAMMA * (float)k.alpha;
    return p;
}

// Fast ASSA setup (degree-2 series, non-exact anchor): one rare branch.
__device__ __forceinline__ AssaPair assa_fast(const Anchor& a, float4 kd, float A, const float* __restrict__ orig,
                                              int64_t gi, int64_t Mpad, float sx, float sy, float sz,
                                              const OpConst& k) {
    AssaPair p;
    const float q = fmaf(a.Ux, kd.x, fmaf(a.Uy, kd.y, fmaf(a.Uz, kd.z, kd.w)));
    const float eps = q * a.invR2;
    const float S = fmaf(eps, fmaf(eps, 1.f / 8.f, -0.25f), 1.f);
    const float Tw = fmaf(eps, fmaf(eps, 3.f / 8.f, -0.5f), 1.f);
    const float eu = fmaf(q * a.inv2Rh, S, a.Eu);
    p.w = (A * (a.h2R * Tw)) * k.two_over_h;
    const float xa = fmaf((float)k.alpha, eu, 0.5f);
    const float t = (xa - 0.5f) + RND_MAGIC;
    const float fl = t - RND_MAGIC;
    p.k = k.alpha * a.na + (__float_as_int(t) - RND_MAGIC_BITS);
    if (fabsf((xa - fl) - 0.5f) > 0.5f - GAMMA * (float)k.alpha) p.k = assa_fix(orig, gi, Mpad, sx, sy, sz, k);
    return p;
}

// 2^x for |x| < 1000 (rare paths): 2^n e^{f ln 2}, f = x - n in [-1/2, 1/2], degree 10 (< 1e-13)
__device__ __forceinline__ double exp2_64(double x) {
    const double magic = 6755399441055744.0;  // 1.5 * 2^52: x + magic rounds x to an integer
    const double tn = x + magic;
    const double n = tn - magic;
    const double z = (x - n) * 0.6931471805599453;
    double p = fma(z, 1.0 / 3628800.0, 1.0 / 362880.0);
    p = fma(z, p, 1.0 / 40320.0);
    p = fma(z, p, 1.0 / 5040.0);
    p = fma(z, p, 1.0 / 720.0);
    p = fma(z, p, 1.0 / 120.0);
    p = fma(z, p, 1.0 / 24.0);
    p = fma(z, p, 1.0 / 6.0);
    p = fma(z, p, 0.5);
    p = fma(z, p, 1.0);
    p = fma(z, p, 1.0);
    const int ni = __double2loint(tn);  // low word of x + magic = n (two's complement)
    return p * __hiloint2double((ni + 1023) << 20, 0);
}

// ---- packed fp32x2 arithmetic (sm_100: FADD2 / FMUL2 / FFMA2)
typedef unsigned long long f2_t;
__device__ __forceinline__ f2_t pk2(float lo, float hi) {
    f2_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void upk2(f2_t v, float& lo, float& hi) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ f2_t mul2(f2_t a, f2_t b) {
    f2_t r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f2_t add2(f2_t a, f2_t b) {
    f2_t r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f2_t sub2(f2_t a, f2_t b) {
    f2_t r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f2_t fma2(f2_t a, f2_t b, f2_t c) {
    f2_t r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
__device__ __forceinline__ float ex2f(float x) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
// g = exp2(K1u u^2) for both halves (two MUFU.EX2)
__device__ __forceinline__ f2_t gauss2(f2_t u2, f2_t K2) {
    float a0, a1;
    upk2(mul2(mul2(u2, K2), u2), a0, a1);
    return pk2(ex2f(a0), ex2f(a1));
}

// ---- factorised Gaussian window ("TAB" fast path).
// For a full window of W = cnt_int samples (W % 4 == 0, W <= 32) centred at
// i = C = W/2, u_i = u_c - m with m = i - C and u_c = u_lo - C in (-1, 0):
//
//   u_i exp2(K u_i^2) = exp2(K u_c^2) * exp2(-2 K u_c)^m * [exp2(K m^2) (u_c - m)]
//                     =       E       *        r^m       *      Q_m(u_c)
//
// Q_m = fma(u_c, c_m, d_m) with the per-operator table c_m = exp2(K m^2),
// d_m = -m c_m (fp64 on the host, each rounded to fp32), i.e. Q_m = c_m (u_c - m).  r^m is a
// geometric chain from the centre (up by r, down by s = 1/r = exp2(2 K u_c)),
// so per pair there are 3 MUFU.EX2 (E, r, s) instead of W, and per sample one
// FFMA (Q), one FMUL (chain) and one FFMA (accumulate), all in f32x2.
//
// r and s multiply into every sample at |m| > 0 (r^m), so a BIASED error in
// them becomes an even-shaped systematic error that the strongly cancelling
// sums of y do not average away (measured: MUFU.EX2 for r, s gave 4e-4
// elementwise at cfg4).  They are therefore evaluated as e^{+-x} =
// C(x^2) +- x S(x^2), x = -2 K ln2 u_c in (-kappa, 0), kappa = -2 K ln2 <= 0.25
// for W >= TAB_MIN, with the Taylor polynomials to x^7 (truncation < 4e-10),
// i.e. to fp32 rounding.  E multiplies the whole pulse and keeps MUFU.EX2.
constexpr int TAB_MIN = 12;
constexpr int TAB_MAX = 32;
struct TabConst {
    f2_t c2[TAB_MAX / 2];  // (c_i, c_{i+1}), i even, i = 0..W-1 (sample index in the window)
    f2_t d2[TAB_MAX / 2];  // (d_i, d_{i+1}) = -(i - C) c_i
    float m2K;             // -2 K1u
    float K;               // K1u
    float kappa;           // -2 K1u ln 2
    int32_t on;            // 1: cnt_int == W, W % 4 == 0, TAB_MIN <= W <= TAB_MAX, degree-2 series path
    int32_t pscale;        // 1: per-pair scale by the unbiased polynomial (wide 1/r spread, set at create)
    float inv_h;           // f_s / v (group radius in samples, union window)
    f2_t g2[11];           // union window: (G_2i, G_2i+1), G_p = 2^{K (p - 11)^2} (k_forward<.., UNION>)
};

// r = exp2(-2 K u_c), s = 1 / r for two pairs (f32x2)
__device__ __forceinline__ void tab_rs(f2_t uc, const TabConst& t, f2_t& r, f2_t& s) {
    const f2_t x = mul2(uc, pk2(t.kappa, t.kappa));
    const f2_t y = mul2(x, x);
    f2_t C = fma2(y, pk2(1.f / 720.f, 1.f / 720.f), pk2(1.f / 24.f, 1.f / 24.f));
    C = fma2(y, C, pk2(0.5f, 0.5f));
    C = fma2(y, C, pk2(1.f, 1.f));
    f2_t S = fma2(y, pk2(1.f / 5040.f, 1.f / 5040.f), pk2(1.f / 120.f, 1.f / 120.f));
    S = fma2(y, S, pk2(1.f / 6.f, 1.f / 6.f));
    S = fma2(y, S, pk2(1.f, 1.f));
    const f2_t xS = mul2(x, S);
    r = add2(C, xS);
    s = sub2(C, xS);
}

// r - 1 and s - 1 (r = exp2(-2K u_c), s = 1/r) for two pairs: the chains P r^m
// multiply by 1 + eps (FFMA P eps + P), so the fp32 rounding of the multiplier is
// relative to |eps| <= 0.3 instead of 1 (the "near-1" form; same cost as FMUL)
__device__ __forceinline__ void tab_rs_eps(f2_t uc, const TabConst& t, f2_t& er, f2_t& es) {
    const f2_t x = mul2(uc, pk2(t.kappa, t.kappa));
    const f2_t y = mul2(x, x);
    f2_t C1 = fma2(y, pk2(1.f / 720.f, 1.f / 720.f), pk2(1.f / 24.f, 1.f / 24.f));
    C1 = fma2(y, C1, pk2(0.5f, 0.5f));
    C1 = mul2(y, C1);  // cosh(x) - 1
    f2_t S = fma2(y, pk2(1.f / 5040.f, 1.f / 5040.f), pk2(1.f / 120.f, 1.f / 120.f));
    S = fma2(y, S, pk2(1.f / 6.f, 1.f / 6.f));
    S = fma2(y, S, pk2(1.f, 1.f));
    const f2_t xS = mul2(x, S);  // sinh(x)
    er = add2(C1, xS);
    es = sub2(C1, xS);
}

// Packed (two pairs) series S(eps) of (sqrt(1+eps)-1)/(eps/2) and T(eps) of
// (1+eps)^-1/2: degree 2 / 2 (SER 0, |eps| <= EPS_SMALL) or 5 / 4 (SER_FAST5,
// |eps| <= EPS_FAST) -- the same polynomials as pair_setup<2> / pair_setup<5>.
template <int DEG>
__device__ __forceinline__ void series2(f2_t eps, f2_t& S, f2_t& Tw) {
    const f2_t one = pk2(1.f, 1.f);
    if (DEG <= 2) {
        S = fma2(eps, fma2(eps, pk2(1.f / 8.f, 1.f / 8.f), pk2(-0.25f, -0.25f)), one);
        Tw = fma2(eps, fma2(eps, pk2(3.f / 8.f, 3.f / 8.f), pk2(-0.5f, -0.5f)), one);
    } else {
        S = fma2(eps, pk2(-21.f / 512.f, -21.f / 512.f), pk2(7.f / 128.f, 7.f / 128.f));
        S = fma2(eps, S, pk2(-5.f / 64.f, -5.f / 64.f));
        S = fma2(eps, S, pk2(1.f / 8.f, 1.f / 8.f));
        S = fma2(eps, S, pk2(-0.25f, -0.25f));
        S = fma2(eps, S, one);
        Tw = fma2(eps, pk2(35.f / 128.f, 35.f / 128.f), pk2(-5.f / 16.f, -5.f / 16.f));
        Tw = fma2(eps, Tw, pk2(3.f / 8.f, 3.f / 8.f));
        Tw = fma2(eps, Tw, pk2(-0.5f, -0.5f));
        Tw = fma2(eps, Tw, one);
    }
}

// Forward accumulate of one pair's W samples into its smem column (lane stride
// 32; ap points at sample n_lo).  P0 = w E; r, s = exp2(-/+2 K u_c).
template <int W>
__device__ __forceinline__ void acc_tab(float* ap, float uc, float P0, float r, float s, const TabConst& t) {
    constexpr int C = W / 2;
    const f2_t U = pk2(uc, uc);
    f2_t P = pk2(P0, P0 * r);  // (P_0, P_1)
    const float r2 = r * r;
#pragma unroll
    for (int i = C; i < W; i += 2) {
        const f2_t Q = fma2(U, t.c2[i / 2], t.d2[i / 2]);
        f2_t acc2 = pk2(ap[i * 32], ap[(i + 1) * 32]);
        acc2 = fma2(P, Q, acc2);
        float v0, v1;
        upk2(acc2, v0, v1);
        ap[i * 32] = v0;
        ap[(i + 1) * 32] = v1;
        P = mul2(P, pk2(r2, r2));
    }
    const float s2 = s * s;
    f2_t Pd = pk2(P0 * s2, P0 * s);  // (P_-2, P_-1)
#pragma unroll
    for (int i = C - 2; i >= 0; i -= 2) {
        const f2_t Q = fma2(U, t.c2[i / 2], t.d2[i / 2]);
        f2_t acc2 = pk2(ap[i * 32], ap[(i + 1) * 32]);
        acc2 = fma2(Pd, Q, acc2);
        float v0, v1;
        upk2(acc2, v0, v1);
        ap[i * 32] = v0;
        ap[(i + 1) * 32] = v1;
        Pd = mul2(Pd, pk2(s2, s2));
    }
}

// Forward accumulate of one pair's W samples into its smem column (lane stride
// 32; ap points at sample n_lo).  P0 = w E; er, es = r - 1, s - 1 with
// r, s = exp2(-/+2 K u_c) (tab_rs_eps): every chain step is P (1 + eps).
template <int W>
__device__ __forceinline__ void acc_tab_eps(float* ap, float uc, float P0, float er, float es, const TabConst& t) {
    constexpr int C = W / 2;

    const f2_t U = pk2(uc, uc);
    f2_t P = pk2(P0, fmaf(P0, er, P0));  // (P_0, P_1)
    const float e2 = fmaf(er, er, 2.f * er);  // r^2 - 1
#pragma unroll
    for (int i = C; i < W; i += 2) {
        const f2_t Q = fma2(U, t.c2[i / 2], t.d2[i / 2]);
        f2_t acc2 = pk2(ap[i * 32], ap[(i + 1) * 32]);
        acc2 = fma2(P, Q, acc2);
        float v0, v1;
        upk2(acc2, v0, v1);
        ap[i * 32] = v0;
        ap[(i + 1) * 32] = v1;
        P = fma2(P, pk2(e2, e2), P);
    }
    const float Pm1 = fmaf(P0, es, P0);
    const float f2 = fmaf(es, es, 2.f * es);  // s^2 - 1
    f2_t Pd = pk2(fmaf(Pm1, es, Pm1), Pm1);  // (P_-2, P_-1)
#pragma unroll
    for (int i = C - 2; i >= 0; i -= 2) {
        const f2_t Q = fma2(U, t.c2[i / 2], t.d2[i / 2]);
        f2_t acc2 = pk2(ap[i * 32], ap[(i + 1) * 32]);
        acc2 = fma2(Pd, Q, acc2);
        float v0, v1;
        upk2(acc2, v0, v1);
        ap[i * 32] = v0;
        ap[(i + 1) * 32] = v1;
        Pd = fma2(Pd, pk2(f2, f2), Pd);
    }
}

// ---- sensor-lane adjoint helpers (gpair_kernels.cu, gpair_assa.cu)
constexpr int STAGE_CELLS = 8;  // cells per staged kernel tile
// Reduce-scatter of 8 per-lane values (one group of 8 kernels) over the warp's 32
// sensors: xor 16 / 8 / 4 halve the value set, xor 2 / 1 finish the sums; lane 4k
// ends with kernel k's sum and writes it to dst[k] (fixed order: deterministic).
template <typename VT>
__device__ __forceinline__ void warp_reduce_scatter8(const VT (&gv)[GROUP], int lane, gacc_t* dst) {
    const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
    gacc_t h4[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const gacc_t keep = b4 ? gv[4 + i] : gv[i], send = b4 ? gv[i] : gv[4 + i];
        h4[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
    gacc_t h2[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const gacc_t keep = b3 ? h4[2 + i] : h4[i], send = b3 ? h4[i] : h4[2 + i];
        h2[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
    gacc_t h1 = (b2 ? h2[1] : h2[0]) + __shfl_xor_sync(0xffffffffu, b2 ? h2[0] : h2[1], 4);
    h1 += __shfl_xor_sync(0xffffffffu, h1, 2);
    h1 += __shfl_xor_sync(0xffffffffu, h1, 1);
    if ((lane & 3) == 0) dst[lane >> 2] = h1;  // lane bits (4, 3, 2) = kernel index
}

// Kernel tile of nc cells into shared memory, kernel pairs interleaved:
// s_kxy[p] = (x0, x1, y0, y1), s_kzw[p] = (z0, z1, w0, w1), plus the group anchors.
__device__ __forceinline__ void stage_kernel_tile(const float4* __restrict__ kd, const float4* __restrict__ grp, int cb,
                                                  int nc, float* s_kxy, float* s_kzw, float4* s_grp) {
    for (int t = threadIdx.x; t < nc * CELL; t += blockDim.x) {
        const float4 v = kd[(int64_t)cb * CELL + t];
        const int pb = (t >> 1) * 4 + (t & 1);
        s_kxy[pb] = v.x;
        s_kxy[pb + 2] = v.y;
        s_kzw[pb] = v.z;
        s_kzw[pb + 2] = v.w;
    }
    if (threadIdx.x < nc * GPC) s_grp[threadIdx.x] = grp[(int64_t)cb * GPC + threadIdx.x];
}

// Sum of the CTA's per-warp kernel sums in warp order -> this sensor group's partial gradient.
__device__ __forceinline__ void write_group_partials(const gacc_t* s_g, int nw, int nc, gacc_t* __restrict__ dst,
                                                     int stride = STAGE_CELLS * CELL) {
    for (int t = threadIdx.x; t < nc * CELL; t += blockDim.x) {
        gacc_t sum = 0;
        for (int w = 0; w < nw; ++w) sum += s_g[w * stride + t];
        dst[t] = sum;
    }
}

}  // namespace gpair
