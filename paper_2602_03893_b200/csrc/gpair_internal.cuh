// gpair_internal.cuh -- shared device helpers of the B200 GPAIR hot path.
//
// Per-pair arithmetic of Eq. 7 with the 3-sigma window
// of P:291, evaluated with a two-level time of flight:
//   * fp64 anchor per (32-kernel cell c, sensor j):  R_cj = |C_c - s_j|,
//     n_a = floor((R/v - t0) f_s),  E = R - v (t0 + n_a/f_s)  (d at sample n_a)
//   * fp32 per-pair offset with q = 2 u.delta + |delta|^2 (u = C_c - s_j,
//     delta = c_i - C_c) and r - R = R (sqrt(1 + q/R^2) - 1) by a degree-5
//     series in eps = q/R^2 (|eps| <= max_eps, checked at create).
//   * window membership |d| < k sigma decided in fp32 unless the window edge
//     is within GAMMA samples of a sample point; then the pair is re-decided
//     bit-identically to the fp64 oracle (same operation order, IEEE fp64).
//   * per-sample values by the Gaussian recurrence
//       g_{m+1} = g_m q_m,  q_{m+1} = q_m c,  c = exp(-h^2/sigma^2)
//     from g_0 = exp(-e0^2/2s^2), q_0 = exp((2 h e0 - h^2)/2s^2), h = v/f_s.
// See DESIGN.md "Kernels" for the error budget of each step.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace gpair {

constexpr int CELL = 32;          // kernels per cell (one warp lane each in the adjoint)
constexpr float GAMMA = 4e-5f;    // ambiguity band of the fp32 window edges [samples]

// Operator constants, computed once on the host in fp64 and passed by value.
struct OpConst {
    double v, fs, t0, ks;  // ks = k * sigma (fp64, same bits as the oracle's k*sigma)
    int32_t Nt, Nd;
    int32_t wmax;          // max in-window count of any pair
    float h;               // v / f_s
    float inv_h;           // f_s / v
    float ksf;             // (float) ks
    float K1;              // -log2(e) / (2 sigma^2):           g0 = exp2(e0^2 K1)
    float K2, K3;          // log2(e) h / sigma^2, -log2(e) h^2/(2 sigma^2): q0 = exp2(e0 K2 + K3)
    float cq;              // exp(-h^2 / sigma^2)
};

// fp64 anchor of a (cell, sensor) pair, reduced to what the per-pair fp32
// arithmetic needs.
struct Anchor {
    float Ux, Uy, Uz;  // 2 (C_c - s_j)
    float E;           // R - v t_{n_a}, in [0, h) up to rounding
    float invR2;       // 1 / R^2
    float inv2R;       // 1 / (2 R)
    float R2;          // R^2
    int32_t na;        // anchor sample index floor((R/v - t0) f_s)
};

__device__ __forceinline__ Anchor make_anchor(float Cx, float Cy, float Cz, float sx, float sy,
                                              float sz, const OpConst& k) {
    double dx = (double)Cx - (double)sx;
    double dy = (double)Cy - (double)sy;
    double dz = (double)Cz - (double)sz;
    double R2 = dx * dx + dy * dy + dz * dz;
    double R = sqrt(R2);
    double na = floor((R / k.v - k.t0) * k.fs);
    double E = R - k.v * (k.t0 + na / k.fs);
    Anchor a;
    a.Ux = (float)(2.0 * dx);
    a.Uy = (float)(2.0 * dy);
    a.Uz = (float)(2.0 * dz);
    a.E = (float)E;
    a.invR2 = (float)(1.0 / R2);
    a.inv2R = (float)(0.5 / R);
    a.R2 = (float)R2;
    a.na = (int32_t)na;
    return a;
}

// Exact (oracle-identical) window of one pair: first and last n with
// |r - v (t0 + n/f_s)| < ks, clipped to [0, N_t).  d(n) = r - v t_n is
// monotone in n (every rounding step is monotone), so the window is found by
// walking from the fp32 guesses g_first / g_last (accurate to +-1 sample).
// r comes from the ORIGINAL fp32 inputs in fp64 with explicit
// round-to-nearest ops (no FMA contraction), exactly like
// oracle/gpair_oracle.c pair_distance() and its membership test, so the
// decision is bit-identical to the oracle's.
__device__ __forceinline__ double exact_d(double r, int n, const OpConst& k) {
    double t = __dadd_rn(k.t0, __ddiv_rn((double)n, k.fs));
    return __dsub_rn(r, __dmul_rn(k.v, t));
}

static __device__ __noinline__ void exact_window(float cx, float cy, float cz, float sx, float sy, float sz,
                                          int g_first, int g_last, const OpConst& k, int& n_lo,
                                          int& cnt) {
    double dx = __dsub_rn((double)cx, (double)sx);
    double dy = __dsub_rn((double)cy, (double)sy);
    double dz = __dsub_rn((double)cz, (double)sz);
    double r2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
    double r = __dsqrt_rn(r2);
    int f = g_first;
    while (exact_d(r, f - 1, k) < k.ks) --f;
    while (!(exact_d(r, f, k) < k.ks)) ++f;
    int l = g_last;
    while (exact_d(r, l + 1, k) > -k.ks) ++l;
    while (!(exact_d(r, l, k) > -k.ks)) --l;
    if (f < 0) f = 0;
    if (l > k.Nt - 1) l = k.Nt - 1;
    n_lo = f;
    cnt = l - f + 1;
    if (cnt < 0) cnt = 0;
}

struct PairWin {
    float e_lo;   // d at the first in-window sample
    float w;      // A / (2 r)
    int32_t n_lo; // first in-window sample
    int32_t cnt;  // number of in-window samples (0 = none)
    int32_t g_first, g_last;  // unclipped fp32 window edges (guesses for exact_window)
    bool amb;     // fp32 edge decision ambiguous -> caller must call exact_window
};

// fp32 per-pair setup from the anchor; kd = (dx, dy, dz, |d|^2) of the kernel
// relative to its cell anchor.
__device__ __forceinline__ PairWin pair_setup(const Anchor& a, float4 kd, float A, const OpConst& k) {
    float q = fmaf(a.Ux, kd.x, fmaf(a.Uy, kd.y, fmaf(a.Uz, kd.z, kd.w)));
    float eps = q * a.invR2;
    // sqrt(1+eps) - 1 = (eps/2) (1 - eps/4 + eps^2/8 - 5eps^3/64 + 7eps^4/128 - 21eps^5/512)
    float poly = fmaf(eps, -21.f / 512.f, 7.f / 128.f);
    poly = fmaf(eps, poly, -5.f / 64.f);
    poly = fmaf(eps, poly, 1.f / 8.f);
    poly = fmaf(eps, poly, -0.25f);
    poly = fmaf(eps, poly, 1.f);
    float dr = (q * a.inv2R) * poly;
    float e = a.E + dr;  // d at sample n_a
    PairWin p;
    p.w = A * 0.5f * rsqrtf(a.R2 + q);
    float alpha = (e - k.ksf) * k.inv_h;  // in-window m satisfy alpha < m < beta
    float beta = (e + k.ksf) * k.inv_h;
    float fa = floorf(alpha), cb = ceilf(beta);
    p.amb = (fabsf(alpha - rintf(alpha)) < GAMMA) || (fabsf(beta - rintf(beta)) < GAMMA);
    int m_lo = (int)fa + 1, m_hi = (int)cb - 1;
    int n_lo = a.na + m_lo, n_hi = a.na + m_hi;
    p.g_first = n_lo;
    p.g_last = n_hi;
    if (n_lo < 0) n_lo = 0;
    if (n_hi > k.Nt - 1) n_hi = k.Nt - 1;
    p.n_lo = n_lo;
    p.cnt = n_hi - n_lo + 1;
    if (p.cnt < 0) p.cnt = 0;
    // offset of the first in-window sample from the anchor sample
    p.e_lo = fmaf(-(float)(n_lo - a.na), k.h, e);
    return p;
}

// After exact_window replaced n_lo, recompute e_lo consistently.
__device__ __forceinline__ float e_at(const Anchor& a, float4 kd, int n, const OpConst& k) {
    float q = fmaf(a.Ux, kd.x, fmaf(a.Uy, kd.y, fmaf(a.Uz, kd.z, kd.w)));
    float eps = q * a.invR2;
    float poly = fmaf(eps, -21.f / 512.f, 7.f / 128.f);
    poly = fmaf(eps, poly, -5.f / 64.f);
    poly = fmaf(eps, poly, 1.f / 8.f);
    poly = fmaf(eps, poly, -0.25f);
    poly = fmaf(eps, poly, 1.f);
    float e = a.E + (q * a.inv2R) * poly;
    return fmaf(-(float)(n - a.na), k.h, e);
}

}  // namespace gpair
