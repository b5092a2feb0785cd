// gpair_kernels.cu -- per-call kernels of the GPAIR hot path.
//
//   k_gather    a2: x = (z + eps)^2 (NPC, Eq. 18) or x as given, into the
//                   spatial order of the cells.
//   k_forward   a3+a4: lane = sensor, warp = 32 sensors, CTA = region of cells
//                   x sensor group.  Kernel parameters are staged in shared
//                   memory and broadcast; each lane accumulates its sensor's
//                   time trace for the region in a private shared-memory
//                   column [sample][32] (conflict-free, no atomics), then the
//                   warp flushes it with 128-byte coalesced stores after an
//                   in-place XOR-swizzled transpose.  Full windows use the
//                   factorised Gaussian (TAB path, gpair_internal.cuh).
//   k_reduce    a5+a6: sums the region partial traces of one sensor in a
//                   fixed order (deterministic), writes y, the residual
//                   delta = y - b and per-sensor loss partials.
//   k_adjoint_t a7: the adjoint with the forward's decomposition (lane =
//                   sensor) on the TAB path; per-sensor-group partial
//                   gradients; k_adj_gather (a8) sums them in order and applies
//                   the fused NPC chain rule (Eq. 19) + Adam, or the clamp step.
//   k_adjoint   a7+a8: lane = kernel, warp = one 32-kernel cell, CTA = region
//                   of cells (every other configuration); residual windows of
//                   32 sensors are staged in shared memory and read per lane
//                   (gather only, no atomics); the epilogue writes g or applies
//                   the update.
#include <algorithm>
#include <cstdlib>

#include "gpair_ctx.h"

namespace gpair {

namespace {


__global__ void k_gather(const float* __restrict__ src, const int32_t* __restrict__ perm, int64_t Mpad,
                         int npc, float eps, float* __restrict__ amp) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= Mpad) return;
    int32_t p = perm[i];
    float a = 0.f;
    if (p >= 0) {
        float v = src[p];
        a = npc ? (v + eps) * (v + eps) : v;
    }
    amp[i] = a;
}

// fp64 polynomial coefficients in the constant bank (DFMA takes them as c[][] operands
// instead of two register moves per use): 1/720, 1/24, 1/2, 1/5040, 1/120, 1/6, 1, 1/8!, 1/9!
__constant__ double kLcfPoly[9] = {1.0 / 720.0, 1.0 / 24.0, 0.5, 1.0 / 5040.0, 1.0 / 120.0, 1.0 / 6.0, 1.0,
                                   1.0 / 40320.0, 1.0 / 362880.0};
// e^{+z} and e^{-z} for |z| <= 0.3: C(z^2) +- z S(z^2), degree 3 in z^2 (truncation < 4e-10,
// and < 4e-12 at the W = 16 bench constants, |z| <= 0.14)
__device__ __forceinline__ void exp_pm64(double z, double& ep, double& em) {
    const double y = z * z;
    double Cc = fma(y, kLcfPoly[0], kLcfPoly[1]);
    Cc = fma(y, Cc, kLcfPoly[2]);
    Cc = fma(y, Cc, kLcfPoly[6]);
    double Sc = fma(y, kLcfPoly[3], kLcfPoly[4]);
    Sc = fma(y, Sc, kLcfPoly[5]);
    Sc = fma(y, Sc, kLcfPoly[6]);
    const double zs = z * Sc;
    ep = Cc + zs;
    em = Cc - zs;
}
// e^{z} for -0.13 <= z <= 0: Taylor degree 6 (truncation < 1e-11)
__device__ __forceinline__ double exp_small64(double z) {
    double p = fma(z, kLcfPoly[0], kLcfPoly[4]);
    p = fma(z, p, kLcfPoly[1]);
    p = fma(z, p, kLcfPoly[5]);
    p = fma(z, p, kLcfPoly[2]);
    p = fma(z, p, kLcfPoly[6]);
    return fma(z, p, kLcfPoly[6]);
}
// 2^{+x} and 2^{-x} for |x| < 1000: x = n + f, n = rint(x), |f| <= 1/2, e^{+-f ln2} = C(z^2) +- z S(z^2)
// (z = f ln 2, degree 4 in z^2: truncation < 1e-11), scaled by 2^{+-n} through the exponent
__device__ __forceinline__ void exp2_pm64(double x, double& ep, double& em) {
    const double magic = 6755399441055744.0;  // 1.5 * 2^52
    const double tn = x + magic;
    const double n = tn - magic;
    const double z = (x - n) * 0.6931471805599453;
    const double y = z * z;
    double Cc = fma(y, kLcfPoly[7], kLcfPoly[0]);
    Cc = fma(y, Cc, kLcfPoly[1]);
    Cc = fma(y, Cc, kLcfPoly[2]);
    Cc = fma(y, Cc, kLcfPoly[6]);
    double Sc = fma(y, kLcfPoly[8], kLcfPoly[3]);
    Sc = fma(y, Sc, kLcfPoly[4]);
    Sc = fma(y, Sc, kLcfPoly[5]);
    Sc = fma(y, Sc, kLcfPoly[6]);
    const double zs = z * Sc;
    const int ni = __double2loint(tn);
    ep = (Cc + zs) * __hiloint2double((1023 + ni) << 20, 0);
    em = (Cc - zs) * __hiloint2double((1023 - ni) << 20, 0);
}
// ------------------------------------------------------------------ forward
#ifndef GPAIR_FWD_MINB
#define GPAIR_FWD_MINB 3
#endif
#ifndef GPAIR_FWD_UNROLL
#define GPAIR_FWD_UNROLL 1
#endif
constexpr int kFwdUnroll = GPAIR_FWD_UNROLL;  // unroll of the 8-kernel group loop
#ifndef GPAIR_FWD_STEP_UNROLL
#define GPAIR_FWD_STEP_UNROLL 1
#endif
// unroll of the fast path's 2-kernel steps in a group: 1 (2: 43.2 ms, 2 with 2 CTAs / SM: 46.7 ms at cfg4;
// profiles/r2/variants_fwd_unroll.txt)
constexpr int kFwdStepUnroll = GPAIR_FWD_STEP_UNROLL;

// Accumulate one pair's WMAX in-window samples into its smem column (lane
// stride 32): packed f32x2, no predicates (the common case).
template <int WMAX>
__device__ __forceinline__ void acc_packed(float* ap, float u_lo, float w, float K1) {
    const f2_t K2 = pk2(K1, K1), W2 = pk2(w, w), step = pk2(-2.f, -2.f);
    f2_t u2 = pk2(u_lo, u_lo - 1.f);
#pragma unroll
    for (int m = 0; m + 1 < WMAX; m += 2) {
        f2_t acc2 = pk2(ap[m * 32], ap[(m + 1) * 32]);
        acc2 = fma2(mul2(W2, u2), gauss2(u2, K2), acc2);
        float v0, v1;
        upk2(acc2, v0, v1);
        ap[m * 32] = v0;
        ap[(m + 1) * 32] = v1;
        u2 = add2(u2, step);
    }
    if (WMAX & 1) {  // odd window length: the last sample alone (exactly WMAX samples are in the window)
        const float um = u_lo - (float)(WMAX - 1);
        ap[(WMAX - 1) * 32] = fmaf(w * um, ex2f((um * K1) * um), ap[(WMAX - 1) * 32]);
    }
}

// Any window length (clipped / exact-edge / general pairs).
template <int WMAX>
__device__ __forceinline__ void acc_generic(float* ap, float u_lo, float w, float K1, int cnt) {
#pragma unroll
    for (int m = 0; m < WMAX; ++m) {
        if (m < cnt) {
            const float um = u_lo - (float)m;
            const float g = ex2f((um * K1) * um);
            ap[m * 32] = fmaf(w * um, g, ap[m * 32]);
        }
    }
    for (int m = WMAX; m < cnt; ++m) {  // only if an exact window exceeds WMAX
        const float um = u_lo - (float)m;
        ap[m * 32] = fmaf(w * um, ex2f((um * K1) * um), ap[m * 32]);
    }
}

template <int WMAX>
__device__ __forceinline__ void acc_pair(float* s_acc_lane, int lo_j, const PairWin& p, float K1) {
    if (p.cnt <= 0) return;
    float* ap = s_acc_lane + (p.n_lo - lo_j) * 32;
    if (p.cnt == WMAX && (WMAX & 1) == 0)
        acc_packed<WMAX>(ap, p.u_lo, p.w, K1);
    else
        acc_generic<WMAX>(ap, p.u_lo, p.w, K1, p.cnt);
}

// cp.async helpers (L1-allocating 4-B and 16-B copies into shared memory)
__device__ __forceinline__ void cp_async_f32(float* dst, const float* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async_16(float* dst, const float4* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit_group() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

constexpr int FWD_STAGE = 6;                                        // cells per double-buffered tile (FAST)
constexpr int FWD_BUF = FWD_STAGE * CELL * 5 + FWD_STAGE * GPC * 4;  // floats per tile buffer

// Register-window union (UNION, W = 16 compact geometries): the 8 pairs of a group are
// evaluated at the 22 positions of their union window in registers and the group's sums
// are added to the lane's column once per position:
//   value(P0 + p) = w (a - tau_p) 2^{K (a - tau_p)^2},  tau_p = p - 11,  a = u_c + k - 3
//                 = G_p * alpha rho^tau_p (tau_p - a) * (-1),  alpha = w 2^{K a^2}, rho = 2^{-2K a},
// with G_p = 2^{K tau_p^2} applied at the group flush (constant per position).  The chains
// rho^tau run from the window centre (tau = 0) outward; k = window start - P0 in [0, 6] (P0 from
// the anchor and the group radius); positions 6..15 lie in every window, the 6 + 6 edge
// positions are masked per pair.  Accumulation: 8 pairs in registers, then one fp32 add per
// group and position into the column (64 groups per 512-kernel region: no split needed).
constexpr int UNION_U = 22;

template <int WMAX, int SER, bool UNION = false>
__global__ void __launch_bounds__(256, GPAIR_FWD_MINB) k_forward(const float4* __restrict__ kd, const float* __restrict__ amp,
                                                 const float4* __restrict__ grp, const float* __restrict__ orig,
                                                 const float* __restrict__ sens, const int32_t* __restrict__ wlo,
                                                 float* __restrict__ partial, int32_t cpr, int32_t ncells,
                                                 int32_t Lf, int64_t Mpad, OpConst k,
                                                 const float4* __restrict__ ksig, const TabConst tab, int32_t split) {
    constexpr bool GEN = SER == SER_GEN;
    // two pairs per setup in f32x2 (exact-integer window length): degree-2 or degree-5 series
    constexpr bool FAST = SER == 0 || SER == SER_FAST5;
    constexpr int SDEG = SER == 0 ? 2 : 5;
    // factorised Gaussian (TabConst): 3 MUFU per pair instead of WMAX
    constexpr bool TABW = FAST && (WMAX % 4 == 0) && WMAX >= TAB_MIN && WMAX <= TAB_MAX;
    extern __shared__ float4 smem4[];
    // FAST: double-buffered parameter tiles of FWD_STAGE cells, filled by cp.async while the
    // previous tile is evaluated; kernel pairs interleaved, s_kxy[p] = (x0, x1, y0, y1),
    // s_kzw[p] = (z0, z1, w0, w1), then amplitudes and the group anchors.
    // Other paths: one synchronous tile of STAGE_CELLS cells (s_kd AoS).
    // double buffering pays when the per-tile evaluation is long (W >= 12); short windows
    // (W = 5, 8) keep one synchronous tile of STAGE_CELLS cells (fewer barriers per kernel)
    constexpr bool DBUF = FAST && WMAX >= 12;
    constexpr int STG = DBUF ? FWD_STAGE : STAGE_CELLS;
    float4* s_kd = smem4;                                   // [STAGE_CELLS*32] (non-FAST)
    float4* s_grp = s_kd + STAGE_CELLS * CELL;              // [STAGE_CELLS*GPC]
    float* s_amp = (float*)(s_grp + STAGE_CELLS * GPC);     // [STAGE_CELLS*32]
    float4* s_ks = (float4*)(s_amp + STAGE_CELLS * CELL);   // [STAGE_CELLS*32] (GEN only)
    float* s_kxy = (float*)s_kd;
    float* s_kzw = s_kxy + STAGE_CELLS * CELL * 2;
    const int nw = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // split-accumulation: the CTA's warps are nsw sensor warps x split kernel subsets; warp
    // (q, sw) accumulates every split-th 8-kernel group of the region for the 32 sensors of
    // sensor warp sw into its own column, and the split columns are summed before the flush:
    // fp32 accumulation chains split times shorter (forward accuracy)
    const int nsw = nw / split, sw = warp % nsw, q = warp / nsw;
    float* s_acc = (DBUF ? (float*)smem4 + 2 * FWD_BUF : (float*)(s_ks + (GEN ? STAGE_CELLS * CELL : 0))) +
                   (size_t)warp * Lf * 32;
    float* s_acc_lane = s_acc + lane;

    const int region = blockIdx.x;
    const int jbase = ((blockIdx.y + k.grp0) * nsw + sw) * 32;
    const int j = jbase + lane;
    const bool jok = j < k.Nd;
    for (int t = lane; t < Lf * 32; t += 32) s_acc[t] = 0.f;
    const int lo_j = jok ? wlo[(int64_t)region * k.Nd + j] : -1;
    float sx = 0.f, sy = 0.f, sz = 0.f;
    if (jok) {
        sx = sens[j];
        sy = sens[k.Nd + j];
        sz = sens[2 * k.Nd + j];
    }
    const int c0 = region * cpr, c1 = min(c0 + cpr, ncells);
    auto issue_tile = [&](int cbs, int buf) {  // FAST: cp.async of one parameter tile into buffer buf
        const int ncs = min(FWD_STAGE, c1 - cbs);
        float* bxy = (float*)smem4 + buf * FWD_BUF;
        float* bzw = bxy + FWD_STAGE * CELL * 2;
        float* bam = bzw + FWD_STAGE * CELL * 2;
        float* bgr = bam + FWD_STAGE * CELL;
        for (int t = threadIdx.x; t < ncs * CELL; t += blockDim.x) {
            const float* src = (const float*)(kd + (int64_t)cbs * CELL + t);
            const int pb = (t >> 1) * 4 + (t & 1);
            cp_async_f32(bxy + pb, src);
            cp_async_f32(bxy + pb + 2, src + 1);
            cp_async_f32(bzw + pb, src + 2);
            cp_async_f32(bzw + pb + 2, src + 3);
            cp_async_f32(bam + t, amp + (int64_t)cbs * CELL + t);
        }
        if (threadIdx.x < ncs * GPC) cp_async_16(bgr + 4 * threadIdx.x, grp + (int64_t)cbs * GPC + threadIdx.x);
    };
    if (DBUF && c0 < c1) issue_tile(c0, 0);
    cp_async_commit_group();
    int stage = 0;
    for (int cb = c0; cb < c1; cb += STG, ++stage) {
        const int nc = min(STG, c1 - cb);
        __syncthreads();  // every warp is done with the previous tile (FAST: buffer (stage + 1) & 1)
        if constexpr (DBUF) {
            if (cb + STG < c1) issue_tile(cb + STG, (stage + 1) & 1);
            cp_async_commit_group();
            cp_async_wait_1();  // this tile's copies (this thread's) have landed
            s_kxy = (float*)smem4 + (stage & 1) * FWD_BUF;
            s_kzw = s_kxy + FWD_STAGE * CELL * 2;
            s_amp = s_kzw + FWD_STAGE * CELL * 2;
            s_grp = (float4*)(s_amp + FWD_STAGE * CELL);
        } else {
            for (int t = threadIdx.x; t < nc * CELL; t += blockDim.x) {
                const float4 v = kd[(int64_t)cb * CELL + t];
                if (FAST) {  // pair-interleaved, as in the double-buffered tiles
                    const int pb = (t >> 1) * 4 + (t & 1);
                    s_kxy[pb] = v.x;
                    s_kxy[pb + 2] = v.y;
                    s_kzw[pb] = v.z;
                    s_kzw[pb + 2] = v.w;
                } else {
                    s_kd[t] = v;
                }
                s_amp[t] = amp[(int64_t)cb * CELL + t];
                if (GEN) s_ks[t] = ksig[(int64_t)cb * CELL + t];
            }
            if (threadIdx.x < nc * GPC) s_grp[threadIdx.x] = grp[(int64_t)cb * GPC + threadIdx.x];
        }
        __syncthreads();
        for (int gq = q; gq < nc * GPC && lo_j >= 0; gq += split) {
            const Anchor a = make_anchor(s_grp[gq], sx, sy, sz, k);
            if constexpr (FAST) {
                if (!__any_sync(__activemask(), a.na == NA_EXACT)) {
                    // union window eligibility: group radius <= 2.5 samples (k in [0, 6]), uniform per group
                    const float dR = s_grp[gq].w * tab.inv_h * 1.0001f + 1e-3f;
                    const bool uni = UNION && dR <= 2.5f;
                    // union start (column index): round(eu + c_lo) + 1 + n_a - lo_j over eu in [Eu - dR, Eu + dR]
                    const int P0 = (int)floorf(a.Eu + k.c_lo - dR + 0.5f) + 1 + (a.na - lo_j);
                    f2_t Su[UNION_U / 2];
#pragma unroll
                    for (int i = 0; i < UNION_U / 2; ++i) Su[i] = 0ull;
                    // Two pairs per step: pair_fast's arithmetic in f32x2 (bit-identical
                    // results), the anchor's per-lane scalars broadcast to both halves.
                    const f2_t Ux = pk2(a.Ux, a.Ux), Uy = pk2(a.Uy, a.Uy), Uz = pk2(a.Uz, a.Uz);
                    const f2_t iR2 = pk2(a.invR2, a.invR2), i2Rh = pk2(a.inv2Rh, a.inv2Rh);
                    const f2_t Eu = pk2(a.Eu, a.Eu), h2R = pk2(a.h2R, a.h2R), clo = pk2(k.c_lo, k.c_lo);
                    const f2_t c8 = pk2(1.f / 8.f, 1.f / 8.f), c4 = pk2(-0.25f, -0.25f), one = pk2(1.f, 1.f);
                    const f2_t c38 = pk2(3.f / 8.f, 3.f / 8.f), c2 = pk2(-0.5f, -0.5f);
                    const f2_t mag = pk2(RND_MAGIC, RND_MAGIC), nmag = pk2(-RND_MAGIC, -RND_MAGIC);
                    const int nrel = a.na - (RND_MAGIC_BITS - 1) - lo_j;  // n_lo - lo_j = bits(t) + nrel
                    const unsigned span = (unsigned)(k.Nt - k.cnt_int);
#pragma unroll kFwdStepUnroll
                    for (int t = 0; t < GROUP; t += 2) {
                        const int li = gq * GROUP + t;
                        const float4 pxy = *(const float4*)(s_kxy + 2 * li), pzw = *(const float4*)(s_kzw + 2 * li);
                        const f2_t kx = pk2(pxy.x, pxy.y), ky = pk2(pxy.z, pxy.w);
                        const f2_t kz = pk2(pzw.x, pzw.y), kw = pk2(pzw.z, pzw.w);
                        const f2_t A2 = *(const f2_t*)(s_amp + li);
                        const f2_t q = fma2(Ux, kx, fma2(Uy, ky, fma2(Uz, kz, kw)));
                        const f2_t eps = mul2(q, iR2);
                        f2_t S, Tw;
                        series2<SDEG>(eps, S, Tw);
                        const f2_t eu = fma2(mul2(q, i2Rh), S, Eu);
                        const f2_t w = mul2(A2, mul2(h2R, Tw));
                        const f2_t x = add2(eu, clo);
                        const f2_t tt = add2(x, mag);
                        const f2_t fl = add2(tt, nmag);
                        const f2_t d = sub2(x, fl);
                        const f2_t ulo = sub2(eu, add2(fl, one));
                        float d0, d1, t0, t1, u0, u1, w0, w1;
                        upk2(d, d0, d1);
                        upk2(tt, t0, t1);
                        upk2(ulo, u0, u1);
                        upk2(w, w0, w1);
                        const int n0 = __float_as_int(t0) + nrel, n1 = __float_as_int(t1) + nrel;
                        const bool bad0 = fabsf(d0) > 0.5f - GAMMA || (unsigned)(n0 + lo_j) > span;
                        const bool bad1 = fabsf(d1) > 0.5f - GAMMA || (unsigned)(n1 + lo_j) > span;
                        const int ku0 = n0 - P0, ku1 = n1 - P0;
                        if (UNION && uni && !(bad0 || bad1) && (unsigned)ku0 <= 6u && (unsigned)ku1 <= 6u) {
                            // a = u_c + k - 3 (|a| < 4); alpha = w 2^{K a^2}; rho = 2^{-2K a}, 1/rho
                            const f2_t uc = add2(ulo, pk2(-(float)(WMAX / 2), -(float)(WMAX / 2)));
                            const f2_t av = add2(uc, pk2((float)(ku0 - 3), (float)(ku1 - 3)));
                            float a0, a1, e0, e1;
                            upk2(av, a0, a1);
                            upk2(mul2(mul2(av, pk2(tab.K, tab.K)), av), e0, e1);
                            float al0, al1;
                            upk2(mul2(w, pk2(ex2f(e0), ex2f(e1))), al0, al1);
                            // e^{+-x}, x = -2K ln2 a (|x| <= 0.56): C(x^2) +- x S(x^2), degree 4 in x^2
                            const f2_t x = mul2(av, pk2(tab.kappa, tab.kappa));
                            const f2_t y = mul2(x, x);
                            f2_t Cc = fma2(y, pk2(1.f / 40320.f, 1.f / 40320.f), pk2(1.f / 720.f, 1.f / 720.f));
                            Cc = fma2(y, Cc, pk2(1.f / 24.f, 1.f / 24.f));
                            Cc = fma2(y, Cc, pk2(0.5f, 0.5f));
                            Cc = fma2(y, Cc, pk2(1.f, 1.f));
                            f2_t Sn = fma2(y, pk2(1.f / 362880.f, 1.f / 362880.f), pk2(1.f / 5040.f, 1.f / 5040.f));
                            Sn = fma2(y, Sn, pk2(1.f / 120.f, 1.f / 120.f));
                            Sn = fma2(y, Sn, pk2(1.f / 6.f, 1.f / 6.f));
                            Sn = fma2(y, Sn, pk2(1.f, 1.f));
                            const f2_t xS = mul2(x, Sn);
                            float rho0, rho1, sig0, sig1;
                            upk2(add2(Cc, xS), rho0, rho1);
                            upk2(sub2(Cc, xS), sig0, sig1);
#pragma unroll
                            for (int h = 0; h < 2; ++h) {
                                const float al = h ? al1 : al0, rho = h ? rho1 : rho0, sig = h ? sig1 : sig0;
                                const float aa = h ? a1 : a0;
                                const int kk = h ? ku1 : ku0;
                                const f2_t na2 = pk2(-aa, -aa);
                                const f2_t r2 = pk2(rho * rho, rho * rho), s2 = pk2(sig * sig, sig * sig);
                                // centre pair i = 5: tau = (-1, 0)
                                const f2_t Xc = pk2(al * sig, al);
                                f2_t X = Xc;
#pragma unroll
                                for (int i = 5; i < UNION_U / 2; ++i) {  // tau = 2i - 11, 2i - 10 upward
                                    if (i > 5) X = mul2(X, r2);
                                    const f2_t D = add2(pk2((float)(2 * i - 11), (float)(2 * i - 10)), na2);
                                    f2_t Xm = X;
                                    if (2 * i + 1 >= WMAX) {  // positions 16..21: in-window iff p < k + 16
                                        float x0, x1;
                                        upk2(X, x0, x1);
                                        Xm = pk2(2 * i - WMAX < kk ? x0 : 0.f, 2 * i + 1 - WMAX < kk ? x1 : 0.f);
                                    }
                                    Su[i] = fma2(D, Xm, Su[i]);
                                }
                                X = Xc;
#pragma unroll
                                for (int i = 4; i >= 0; --i) {  // downward
                                    X = mul2(X, s2);
                                    const f2_t D = add2(pk2((float)(2 * i - 11), (float)(2 * i - 10)), na2);
                                    f2_t Xm = X;
                                    if (2 * i < 6) {  // positions 0..5: in-window iff p >= k
                                        float x0, x1;
                                        upk2(X, x0, x1);
                                        Xm = pk2(2 * i >= kk ? x0 : 0.f, 2 * i + 1 >= kk ? x1 : 0.f);
                                    }
                                    Su[i] = fma2(D, Xm, Su[i]);
                                }
                            }
                        } else if (!(bad0 || bad1)) {
                            if (TABW && tab.on) {
                                // u_c = u_lo - C (exact), E = exp2(K u_c^2), r = exp2(-2K u_c), s = 1/r
                                const f2_t uc = add2(ulo, pk2(-(float)(WMAX / 2), -(float)(WMAX / 2)));
                                f2_t r2, s2;
                                if (tab.pscale)
                                    tab_rs_eps(uc, tab, r2, s2);  // r - 1, s - 1 (near-1 chains)
                                else
                                    tab_rs(uc, tab, r2, s2);
                                float uc0, uc1, p0, p1, r0, r1, q0, q1;
                                upk2(uc, uc0, uc1);
                                if (tab.pscale) {
                                    // per-pair scale in fp32 with few roundings: w = A (h/2R)(1 + (T - 1)),
                                    // E = 2^{K u_c^2} by a degree-5 polynomial (|z| <= 0.13, unbiased)
                                    const f2_t z = mul2(mul2(mul2(uc, pk2(tab.K, tab.K)), uc), pk2(0.69314718f, 0.69314718f));
                                    f2_t ep = fma2(z, pk2(1.f / 120.f, 1.f / 120.f), pk2(1.f / 24.f, 1.f / 24.f));
                                    ep = fma2(z, ep, pk2(1.f / 6.f, 1.f / 6.f));
                                    ep = fma2(z, ep, pk2(0.5f, 0.5f));
                                    ep = fma2(z, ep, pk2(1.f, 1.f));
                                    ep = fma2(z, ep, pk2(1.f, 1.f));
                                    const f2_t wq = fma2(h2R, sub2(Tw, one), h2R);
                                    upk2(mul2(mul2(A2, ep), wq), p0, p1);
                                } else {  // E by MUFU.EX2 (the compact geometries of cfg2-4)
                                    float e0, e1;
                                    upk2(mul2(mul2(uc, pk2(tab.K, tab.K)), uc), e0, e1);
                                    upk2(mul2(w, pk2(ex2f(e0), ex2f(e1))), p0, p1);
                                }
                                upk2(r2, r0, r1);
                                upk2(s2, q0, q1);
                                if (tab.pscale) {  // wide geometries: the near-1 chains (acc_tab_eps)
                                    acc_tab_eps<TABW ? WMAX : 4>(s_acc_lane + n0 * 32, uc0, p0, r0, q0, tab);
                                    acc_tab_eps<TABW ? WMAX : 4>(s_acc_lane + n1 * 32, uc1, p1, r1, q1, tab);
                                } else {
                                    acc_tab<TABW ? WMAX : 4>(s_acc_lane + n0 * 32, uc0, p0, r0, q0, tab);
                                    acc_tab<TABW ? WMAX : 4>(s_acc_lane + n1 * 32, uc1, p1, r1, q1, tab);
                                }
                            } else {
                                acc_packed<WMAX>(s_acc_lane + n0 * 32, u0, w0, k.K1u);
                                acc_packed<WMAX>(s_acc_lane + n1 * 32, u1, w1, k.K1u);
                            }
                        } else {  // rare: exact window edges and/or record clipping
                            float e0, e1;
                            upk2(eu, e0, e1);
                            const int64_t gi = (int64_t)cb * CELL + li;
                            PairWin p;
                            p.w = w0;
                            p.n_lo = n0 + lo_j;
                            p.u_lo = u0;
                            p.cnt = k.cnt_int;
                            if (bad0)
                                p = pair_fix(p, e0, a.na, fabsf(d0) > 0.5f - GAMMA, orig, gi, Mpad, sx, sy, sz,
                                             k.cnt_int, k);
                            acc_pair<WMAX>(s_acc_lane, lo_j, p, k.K1u);
                            p.w = w1;
                            p.n_lo = n1 + lo_j;
                            p.u_lo = u1;
                            p.cnt = k.cnt_int;
                            if (bad1)
                                p = pair_fix(p, e1, a.na, fabsf(d1) > 0.5f - GAMMA, orig, gi + 1, Mpad, sx, sy, sz,
                                             k.cnt_int, k);
                            acc_pair<WMAX>(s_acc_lane, lo_j, p, k.K1u);
                        }
                    }
                    if (UNION && uni) {  // the group's union sums -> column (value = -G_p S_p), fixed order
#pragma unroll
                        for (int i = 0; i < UNION_U / 2; ++i) {
                            const int p0 = P0 + 2 * i;
                            float v0, v1, g0, g1;
                            upk2(Su[i], v0, v1);
                            upk2(tab.g2[i], g0, g1);
                            if ((unsigned)p0 < (unsigned)Lf) s_acc_lane[p0 * 32] = fmaf(-g0, v0, s_acc_lane[p0 * 32]);
                            if ((unsigned)(p0 + 1) < (unsigned)Lf)
                                s_acc_lane[(p0 + 1) * 32] = fmaf(-g1, v1, s_acc_lane[(p0 + 1) * 32]);
                        }
                    }
                    continue;
                }
            }
            const float4* kdg = s_kd + gq * GROUP;
            const float* ampg = s_amp + gq * GROUP;
#pragma unroll kFwdUnroll
            for (int t = 0; t < GROUP; ++t) {
                const int li = gq * GROUP + t;
                const int64_t gi = (int64_t)cb * CELL + li;
                PairWin p;
                float K1 = k.K1u;
                const int pb = (li >> 1) * 4 + (li & 1);
                const float4 kdt = FAST ? make_float4(s_kxy[pb], s_kxy[pb + 2], s_kzw[pb], s_kzw[pb + 2]) : kdg[t];
                if (GEN) {
                    const float4 ks4 = s_ks[li];
                    p = pair_gen(a, kdt, ampg[t], ks4, orig, gi, Mpad, sx, sy, sz, k);
                    K1 = ks4.y;
                } else {
                    p = pair_setup<(SER == 0 || GEN) ? 2 : 5>(a, kdt, ampg[t], orig, gi, Mpad, sx, sy, sz, k);
                }
                acc_pair<WMAX>(s_acc_lane, lo_j, p, K1);
            }
        }
    }
    if (split > 1) {  // sum the split columns of each sensor warp into q = 0's, in fixed order
        __syncthreads();
        float* base = s_acc - (size_t)warp * Lf * 32;  // column of warp 0
        for (int r = q; r < Lf; r += split) {
            float v = 0.f;
            for (int qq = 0; qq < split; ++qq) v += base[((size_t)(qq * nsw + sw) * Lf + r) * 32 + lane];
            base[((size_t)sw * Lf + r) * 32 + lane] = v;
        }
        __syncthreads();
        if (q != 0) return;
    }
    __syncwarp();
    // flush: per 32-row block, in-place XOR-swizzled transpose then coalesced stores
    // sensor-major partials [N_d][regions][Lf]: the reducer streams each
    // sensor's partials contiguously
    const size_t jstride = (size_t)gridDim.x * Lf;
    float* dst = partial + (size_t)jbase * jstride + (size_t)region * Lf;
    for (int m0 = 0; m0 < Lf; m0 += 32) {
        const int rows = min(32, Lf - m0);  // 32, or a 16-row tail (Lf is a multiple of 16)
        float v[32];
#pragma unroll
        for (int t = 0; t < 32; ++t) v[t] = (t < rows) ? s_acc[(m0 + t) * 32 + lane] : 0.f;
        __syncwarp();
#pragma unroll
        for (int t = 0; t < 32; ++t)
            if (t < rows) s_acc[(m0 + t) * 32 + (lane ^ t)] = v[t];
        __syncwarp();
        for (int jj = 0; jj < 32; ++jj) {
            if (jbase + jj < k.Nd && lane < rows)
                dst[(size_t)jj * jstride + m0 + lane] = s_acc[(m0 + lane) * 32 + (jj ^ lane)];
        }
    }
}

// ------------------------------------------------------------------ reduce
// One CTA per sensor j.  The region partials of j are visited in the
// per-sensor list sorted by window start (built at create, gpair_setup.cu);
// warp w takes a contiguous block of the list, so its rows cover only
// [lo(first), lo(last) + Lf): a private fp64 smem copy of just that span
// (sum over warps ~ live range + nw Lf, not nw x live range).  Lane = samples
// l and l + 32 of a row: two aligned 128-B loads per row, every DRAM sector
// read once, RED_U rows in flight per warp.  The overlapping copies are summed
// in warp order (deterministic, no atomics).  Fuses the near-field rows, y,
// the residual delta = y - b and one fp64 loss partial per sensor.
#ifndef GPAIR_RED_U
#define GPAIR_RED_U 8
#endif
#ifndef GPAIR_RED_MINB
#define GPAIR_RED_MINB 2
#endif
constexpr int RED_U = GPAIR_RED_U;  // rows in flight per warp
constexpr int RED_WARPS = 16; // warps per CTA

__device__ __forceinline__ int red_lower_bound(const int2* e, int n, int v) {
    int a = 0, b = n;
    while (a < b) {
        const int m = (a + b) >> 1;
        if (e[m].x < v) a = m + 1; else b = m;
    }
    return a;
}

__global__ void __launch_bounds__(32 * RED_WARPS, GPAIR_RED_MINB) k_reduce(const float* __restrict__ partial,
                                                              const int2* __restrict__ ent, int32_t nregions,
                                                              int32_t Lf, OpConst k, float* __restrict__ y,
                                                              const float* __restrict__ b, float* __restrict__ delta,
                                                              double* __restrict__ loss_part,
                                                              const int32_t* __restrict__ near_row,
                                                              const double* __restrict__ ynear) {
    extern __shared__ double s_copy[];
    __shared__ int s_k0;
    __shared__ int s_base[RED_WARPS], s_len[RED_WARPS], s_off[RED_WARPS];
    __shared__ double s_red[RED_WARPS];
    const int j = blockIdx.x + k.j0;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int2* e = ent + (int64_t)j * nregions;
    if (threadIdx.x == 0) s_k0 = red_lower_bound(e, nregions, 0);  // first non-empty window
    __syncthreads();
    const int k0 = s_k0;
    const int per_warp = (nregions - k0 + RED_WARPS - 1) / RED_WARPS;
    const int kb = k0 + warp * per_warp, ke = min(kb + per_warp, nregions);
    if (lane == 0) {
        const int base = kb < ke ? e[kb].x : 0;
        s_base[warp] = base;
        s_len[warp] = kb < ke ? min(e[ke - 1].x + Lf, k.Nt) - base : 0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int o = 0;
        for (int w = 0; w < RED_WARPS; ++w) {
            s_off[w] = o;
            o += s_len[w];
        }
    }
    __syncthreads();
    const int base = s_base[warp], len = s_len[warp];
    double* mine = s_copy + s_off[warp];
    for (int t = lane; t < len; t += 32) mine[t] = 0.0;
    __syncwarp();
    const float* pj = partial + (size_t)j * nregions * Lf;
    for (int kk = kb; kk < ke; kk += 32) {
        const int cnt = min(32, ke - kk);
        const int2 my = lane < cnt ? e[kk + lane] : make_int2(0, 0);
        for (int u = 0; u < cnt; u += RED_U) {
            float v0[RED_U], v1[RED_U];
#pragma unroll
            for (int q = 0; q < RED_U; ++q) {
                const int r = __shfl_sync(0xffffffffu, my.y, (u + q) & 31);
                const float* row = pj + (size_t)r * Lf;
                const bool ok = u + q < cnt;
                v0[q] = (ok && lane < Lf) ? row[lane] : 0.f;
                v1[q] = (ok && lane + 32 < Lf) ? row[lane + 32] : 0.f;
            }
#pragma unroll
            for (int q = 0; q < RED_U; ++q) {
                if (u + q >= cnt) break;
                const int t0 = __shfl_sync(0xffffffffu, my.x, (u + q) & 31) - base + lane;
                if (lane < Lf && t0 < len) mine[t0] += (double)v0[q];
                if (lane + 32 < Lf && t0 + 32 < len) mine[t0 + 32] += (double)v1[q];
            }
            for (int q0 = 64; q0 < Lf; q0 += 32) {  // rows longer than 64 samples
#pragma unroll 1
                for (int q = 0; q < RED_U && u + q < cnt; ++q) {
                    const int lo = __shfl_sync(0xffffffffu, my.x, (u + q) & 31);
                    const int r = __shfl_sync(0xffffffffu, my.y, (u + q) & 31);
                    const int t = lo - base + q0 + lane;
                    if (q0 + lane < Lf && t < len) mine[t] += (double)pj[(size_t)r * Lf + q0 + lane];
                }
            }
        }
    }
    __syncthreads();
    double lsum = 0.0;
    const int64_t row = (int64_t)j * k.Nt;
    const int nrow = near_row ? near_row[j] : -1;  // near-field rows (row f4, gpair_near.cu)
    for (int n = threadIdx.x; n < k.Nt; n += blockDim.x) {
        double ys = 0.0;
        for (int w = 0; w < RED_WARPS; ++w) {
            const int t = n - s_base[w];
            if (t >= 0 && t < s_len[w]) ys += s_copy[s_off[w] + t];
        }
        if (nrow >= 0) ys += ynear[(int64_t)nrow * k.Nt + n];
        const float yv = (float)ys;
        if (y) y[row + n] = yv;
        if (b) {
            const float dv = yv - b[row + n];
            delta[row + n] = dv;
            lsum += (double)dv * (double)dv;
        }
    }
    if (b) {
        for (int o = 16; o > 0; o >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
        if (lane == 0) s_red[warp] = lsum;
        __syncthreads();
        if (threadIdx.x == 0) {
            double sacc = 0.0;
            for (int w = 0; w < RED_WARPS; ++w) sacc += s_red[w];
            loss_part[j] = sacc;
        }
    }
}

// residual + loss partials for world > 1 (y already all-reduced)
__global__ void k_residual(const float* __restrict__ y, const float* __restrict__ b, int32_t Nt,
                           float* __restrict__ delta, double* __restrict__ loss_part, int32_t j0) {
    const int j = blockIdx.x + j0;
    const int64_t row = (int64_t)j * Nt;
    double lsum = 0.0;
    for (int n = threadIdx.x; n < Nt; n += blockDim.x) {
        float dv = y[row + n] - b[row + n];
        delta[row + n] = dv;
        lsum += (double)dv * (double)dv;
    }
    __shared__ double s_red[32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int o = 16; o > 0; o >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
    if (lane == 0) s_red[warp] = lsum;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += s_red[w];
        loss_part[j] = s;
    }
}

__global__ void k_loss(const double* __restrict__ part, int32_t n, double inv_N, const double* __restrict__ reg,
                       int32_t n_reg, double lam, float* out) {
    __shared__ double s[1024], r[1024];
    double a = 0.0, b = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) a += part[i];
    for (int i = threadIdx.x; i < n_reg; i += blockDim.x) b += reg[i];
    s[threadIdx.x] = a;
    r[threadIdx.x] = b;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if ((int)threadIdx.x < o) {
            s[threadIdx.x] += s[threadIdx.x + o];
            r[threadIdx.x] += r[threadIdx.x + o];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) out[0] = (float)(s[0] * inv_N + lam * r[0]);  // Eq. 23: data term + lam R_VCR
}

// ------------------------------------------------------------------ adjoint
constexpr int MODE_COUNT = 3;

template <int WMAX, int SER, int MODE>
__global__ void __launch_bounds__(256) k_adjoint(const float4* __restrict__ kd, const float4* __restrict__ grp,
                                                 const float* __restrict__ orig, const int32_t* __restrict__ perm,
                                                 const float* __restrict__ sens, const int32_t* __restrict__ wlo,
                                                 const float* __restrict__ resid, int32_t cpr, int32_t ncells,
                                                 int32_t La, int64_t Mpad, OpConst k, EpiParams ep,
                                                 unsigned long long* count, const float4* __restrict__ ksig) {
    constexpr bool GEN = SER == SER_GEN;
    extern __shared__ float4 smem4[];
    Anchor* s_anc = (Anchor*)smem4;                          // [nw][GPC][33]
    const int nw = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float4* s_sen = (float4*)(s_anc + nw * GPC * 33);       // [32] batch sensor positions
    int32_t* s_wlo = (int32_t*)(s_sen + 32);                 // [32]
    float* s_res = (float*)(s_wlo + 32);                     // [32][La]

    const int cid = blockIdx.x * cpr + warp;
    const bool cok = (warp < cpr) && (cid < ncells);
    const int64_t gi = (int64_t)cid * CELL + lane;
    float4 d4 = make_float4(0.f, 0.f, 0.f, 0.f);
    if (cok) d4 = kd[gi];
    float4 ks4 = make_float4(0.f, k.K1u, 0.f, 0.f);
    if (GEN && cok) ks4 = ksig[gi];
    const float K1 = ks4.y;
    const Anchor* my_anc = s_anc + (warp * GPC + lane / GROUP) * 33;
    float acc = 0.f;
    unsigned long long npairs = 0;
    const bool real = cok && perm[gi] >= 0;
    for (int jb = 0; jb < k.Nd; jb += 32) {
        const int nj = min(32, k.Nd - jb);
        __syncthreads();
        if (threadIdx.x < 32) s_wlo[threadIdx.x] = threadIdx.x < nj ? wlo[(int64_t)blockIdx.x * k.Nd + jb + threadIdx.x] : -1;
        if (threadIdx.x < nj) {
            const int js = jb + threadIdx.x;
            s_sen[threadIdx.x] = make_float4(sens[js], sens[k.Nd + js], sens[2 * k.Nd + js], 0.f);
        }
        if (cok && lane < nj) {
            const int j = jb + lane;
            const float sx = sens[j], sy = sens[k.Nd + j], sz = sens[2 * k.Nd + j];
#pragma unroll
            for (int gq = 0; gq < GPC; ++gq)
                s_anc[(warp * GPC + gq) * 33 + lane] = make_anchor(grp[(int64_t)cid * GPC + gq], sx, sy, sz, k);
        }
        __syncthreads();
        if (MODE != MODE_COUNT) {
            // warp per sensor row, lane per sample: coalesced row segments, no division
            for (int jj = warp; jj < 32; jj += nw) {
                const int lo = s_wlo[jj];
                const float* src = resid + (int64_t)(jb + jj) * k.Nt;
                float* dstr = s_res + jj * La;
                for (int m = lane; m < La; m += 32) {
                    const int n = lo + m;
                    dstr[m] = (lo >= 0 && n < k.Nt) ? src[n] : 0.f;
                }
            }
            __syncthreads();
        }
        if (!cok) continue;
        float accb = 0.f;
        for (int jj = 0; jj < nj; ++jj) {
            const int lo = s_wlo[jj];
            if (lo < 0) continue;
            const float4 sp = s_sen[jj];
            const Anchor a = my_anc[jj];
            PairWin p;
            if (GEN)
                p = pair_gen(a, d4, 1.f, ks4, orig, gi, Mpad, sp.x, sp.y, sp.z, k);
            else if (SER == 0 && a.na != NA_EXACT)
                p = pair_fast(a, d4, 1.f, orig, gi, Mpad, sp.x, sp.y, sp.z, k);
            else
                p = pair_setup<(SER == 0 || GEN) ? 2 : 5>(a, d4, 1.f, orig, gi, Mpad, sp.x, sp.y, sp.z, k);
            if (p.cnt <= 0) continue;
            if (MODE == MODE_COUNT) {
                npairs += real ? (unsigned long long)p.cnt : 0ull;
                continue;
            }
            const float* rp = s_res + jj * La + (p.n_lo - lo);
            float part = 0.f;
            if (p.cnt == WMAX && (WMAX & 1) == 0) {  // packed pairs, no predicates
                const f2_t K2 = pk2(K1, K1), step = pk2(-2.f, -2.f);
                f2_t u2 = pk2(p.u_lo, p.u_lo - 1.f);
                f2_t part2 = 0ull;
#pragma unroll
                for (int m = 0; m < WMAX; m += 2) {
                    part2 = fma2(mul2(u2, gauss2(u2, K2)), pk2(rp[m], rp[m + 1]), part2);
                    u2 = add2(u2, step);
                }
                float p0, p1;
                upk2(part2, p0, p1);
                part = p0 + p1;
            } else {
#pragma unroll
                for (int m = 0; m < WMAX; ++m) {
                    if (m < p.cnt) {
                        const float um = p.u_lo - (float)m;
                        const float g = ex2f((um * K1) * um);
                        part = fmaf(um * g, rp[m], part);
                    }
                }
                for (int m = WMAX; m < p.cnt; ++m) {
                    const float um = p.u_lo - (float)m;
                    part = fmaf(um * ex2f((um * K1) * um), rp[m], part);
                }
            }
            accb = fmaf(p.w, part, accb);
        }
        acc += accb;
    }
    if (!cok) return;
    if (MODE == MODE_COUNT) {
        for (int o = 16; o > 0; o >>= 1) npairs += __shfl_xor_sync(0xffffffffu, npairs, o);
        if (lane == 0) atomicAdd(count, npairs);
        return;
    }
    const int32_t ic = perm[gi];
    if (ic < 0) return;
    adjoint_epilogue<MODE>(acc, ic, ep);
}

// ------------------------------------------------------------------ adjoint, TAB path, sensor lanes
// The adjoint with the forward's decomposition: lane = sensor j, warp = 32
// sensors, CTA = adjoint region of cells x 256 sensors (blockIdx.y = sensor
// group).  Each lane stages its sensor's residual window [lo_j, lo_j + La) as
// a private smem column [t][32] (conflict-free), keeps the fp64 anchor of the
// current 8-kernel group in registers, sets up two kernels per step in f32x2
// (kernel parameters broadcast from smem) and evaluates
//   g_ij = w E sum_m r^m Q_m(u_c) delta_j[n_c + m]
// with two Horner chains (gpair_internal.cuh TabConst).  The 8 per-lane
// values of a group are summed over the warp's 32 sensors by a reduce-scatter
// of shuffles (lane 4k ends with kernel k), the CTA's warps are summed in
// smem in a fixed order, and each sensor group writes its partial gradient
// gpart[group][i]; k_adj_gather sums the groups in order and applies the
// epilogue (deterministic, no atomics).
#ifndef GPAIR_ADJT_DBL
#define GPAIR_ADJT_DBL 1
#endif
#ifndef GPAIR_ADJT_MINB
#define GPAIR_ADJT_MINB 2
#endif
constexpr int ADJT_DBL = GPAIR_ADJT_DBL;  // 1: doubled residual column (one LDS.64 per sample pair)

template <int W, int SDEG>
__global__ void __launch_bounds__(256, GPAIR_ADJT_MINB) k_adjoint_t(const float4* __restrict__ kd, const float4* __restrict__ grp,
                                                     const float* __restrict__ orig, const float* __restrict__ sens,
                                                     const int32_t* __restrict__ wlo, const float* __restrict__ resid,
                                                     gacc_t* __restrict__ gpart, int32_t cpr, int32_t ncells,
                                                     int32_t La, int64_t Mpad, OpConst k, const TabConst tab) {
    constexpr int C = W / 2;
    extern __shared__ float4 smem4[];
    // kernel pairs interleaved: s_kxy[p] = (x0, x1, y0, y1), s_kzw[p] = (z0, z1, w0, w1)
    float* s_kxy = (float*)smem4;
    float* s_kzw = s_kxy + STAGE_CELLS * CELL * 2;
    float4* s_grp = (float4*)(s_kzw + STAGE_CELLS * CELL * 2);  // [STAGE_CELLS*GPC]
    const int nw = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    gacc_t* s_g = (gacc_t*)(s_grp + STAGE_CELLS * GPC);  // [nw][STAGE_CELLS*CELL] per-warp kernel sums
    // this warp's residual column [La][32] (ADJT_DBL: [La][32] float2 (delta_t, delta_{t+1}))
    float* s_col = (float*)(s_g + nw * STAGE_CELLS * CELL) + (size_t)warp * La * 32 * (1 + ADJT_DBL);
    float* col = s_col + lane;
    f2_t* col2 = (f2_t*)s_col + lane;

    const int region = blockIdx.x;
    const int c0 = region * cpr, c1 = min(c0 + cpr, ncells);
    if (c0 < c1) stage_kernel_tile(kd, grp, c0, min(STAGE_CELLS, c1 - c0), s_kxy, s_kzw, s_grp);
    const int j = ((blockIdx.y + k.grp0) * nw + warp) * 32 + lane;
    const bool jok = j < k.Nd;
    const int lo_j = jok ? wlo[(int64_t)region * k.Nd + j] : -1;
    float sx = 0.f, sy = 0.f, sz = 0.f;
    if (jok) {
        sx = sens[j];
        sy = sens[k.Nd + j];
        sz = sens[2 * k.Nd + j];
    }
    {
        const float* src = resid + (int64_t)j * k.Nt;
        float prev = (lo_j >= 0 && lo_j < k.Nt) ? src[lo_j] : 0.f;
        for (int t = 0; t < La; ++t) {
            const int n = lo_j + t;
            if (ADJT_DBL) {
                const float nxt = (lo_j >= 0 && n + 1 < k.Nt) ? src[n + 1] : 0.f;
                col2[t * 32] = pk2(prev, nxt);
                prev = nxt;
            } else {
                col[t * 32] = (lo_j >= 0 && n < k.Nt) ? src[n] : 0.f;
            }
        }
    }
    const f2_t c8 = pk2(1.f / 8.f, 1.f / 8.f), c4 = pk2(-0.25f, -0.25f), one = pk2(1.f, 1.f);
    const f2_t c38 = pk2(3.f / 8.f, 3.f / 8.f), c2 = pk2(-0.5f, -0.5f);
    const f2_t clo = pk2(k.c_lo, k.c_lo), mag = pk2(RND_MAGIC, RND_MAGIC), nmag = pk2(-RND_MAGIC, -RND_MAGIC);
    const unsigned span = (unsigned)(k.Nt - k.cnt_int);
    for (int cb = c0; cb < c1; cb += STAGE_CELLS) {
        const int nc = min(STAGE_CELLS, c1 - cb);
        if (cb != c0) {  // the first tile was staged with the residual columns
            __syncthreads();  // every warp is done with the previous tile and its s_g sums
            stage_kernel_tile(kd, grp, cb, nc, s_kxy, s_kzw, s_grp);
        }
        __syncthreads();
        for (int gq = 0; gq < nc * GPC; ++gq) {
            const Anchor a = make_anchor(s_grp[gq], sx, sy, sz, k);
            float gv[GROUP];
            const bool exact_grp = __any_sync(0xffffffffu, a.na == NA_EXACT);
            const f2_t Ux = pk2(a.Ux, a.Ux), Uy = pk2(a.Uy, a.Uy), Uz = pk2(a.Uz, a.Uz);
            const f2_t iR2 = pk2(a.invR2, a.invR2), i2Rh = pk2(a.inv2Rh, a.inv2Rh);
            const f2_t Eu = pk2(a.Eu, a.Eu), h2R = pk2(a.h2R, a.h2R);
            const int nrel = a.na - (RND_MAGIC_BITS - 1) - lo_j;  // n_lo - lo_j = bits(tt) + nrel
#pragma unroll
            for (int t = 0; t < GROUP; t += 2) {
                const int li = gq * GROUP + t;
                float g0 = 0.f, g1 = 0.f;
                bool rare = exact_grp;
                if (!exact_grp) {
                    const float4 pxy = *(const float4*)(s_kxy + 2 * li), pzw = *(const float4*)(s_kzw + 2 * li);
                    const f2_t kx = pk2(pxy.x, pxy.y), ky = pk2(pxy.z, pxy.w);
                    const f2_t kz = pk2(pzw.x, pzw.y), kw = pk2(pzw.z, pzw.w);
                    const f2_t q = fma2(Ux, kx, fma2(Uy, ky, fma2(Uz, kz, kw)));
                    const f2_t eps = mul2(q, iR2);
                    f2_t S, Tw;
                    series2<SDEG>(eps, S, Tw);
                    const f2_t eu = fma2(mul2(q, i2Rh), S, Eu);
                    const f2_t w = mul2(h2R, Tw);
                    const f2_t x = add2(eu, clo);
                    const f2_t tt = add2(x, mag);
                    const f2_t fl = add2(tt, nmag);
                    const f2_t d = sub2(x, fl);
                    const f2_t ulo = sub2(eu, add2(fl, one));
                    float d0, d1, t0, t1;
                    upk2(d, d0, d1);
                    upk2(tt, t0, t1);
                    const int n0 = __float_as_int(t0) + nrel, n1 = __float_as_int(t1) + nrel;
                    const bool bad0 = fabsf(d0) > 0.5f - GAMMA || (unsigned)(n0 + lo_j) > span;
                    const bool bad1 = fabsf(d1) > 0.5f - GAMMA || (unsigned)(n1 + lo_j) > span;
                    rare = bad0 || bad1;
                    if (!rare && lo_j >= 0) {
                        const f2_t uc = add2(ulo, pk2(-(float)C, -(float)C));
                        f2_t r2p, s2p;
                        tab_rs(uc, tab, r2p, s2p);
                        float e0, e1, P00, P01, uc0, uc1, r0, r1, s0, s1;
                        upk2(mul2(mul2(uc, pk2(tab.K, tab.K)), uc), e0, e1);
                        upk2(mul2(w, pk2(ex2f(e0), ex2f(e1))), P00, P01);
                        upk2(uc, uc0, uc1);
                        upk2(r2p, r0, r1);
                        upk2(s2p, s0, s1);
                        const int rp0 = n0, rp1 = n1;  // window starts in the column
                        auto ldp = [&](int r0, int i) -> f2_t {
                            return ADJT_DBL ? col2[(r0 + i) * 32] : pk2(col[(r0 + i) * 32], col[(r0 + i + 1) * 32]);
                        };
                        const f2_t U0 = pk2(uc0, uc0), U1 = pk2(uc1, uc1);
                        const float rr0 = r0 * r0, ss0 = s0 * s0, rr1 = r1 * r1, ss1 = s1 * s1;
                        f2_t Q0 = fma2(U0, tab.c2[(W - 2) / 2], tab.d2[(W - 2) / 2]);
                        f2_t Q1 = fma2(U1, tab.c2[(W - 2) / 2], tab.d2[(W - 2) / 2]);
                        f2_t Sh0 = mul2(Q0, ldp(rp0, W - 2));
                        f2_t Sh1 = mul2(Q1, ldp(rp1, W - 2));
#pragma unroll
                        for (int i = W - 4; i >= C; i -= 2) {
                            Q0 = fma2(U0, tab.c2[i / 2], tab.d2[i / 2]);
                            Q1 = fma2(U1, tab.c2[i / 2], tab.d2[i / 2]);
                            Sh0 = fma2(Sh0, pk2(rr0, rr0), mul2(Q0, ldp(rp0, i)));
                            Sh1 = fma2(Sh1, pk2(rr1, rr1), mul2(Q1, ldp(rp1, i)));
                        }
                        Q0 = fma2(U0, tab.c2[0], tab.d2[0]);
                        Q1 = fma2(U1, tab.c2[0], tab.d2[0]);
                        f2_t Th0 = mul2(Q0, ldp(rp0, 0));
                        f2_t Th1 = mul2(Q1, ldp(rp1, 0));
#pragma unroll
                        for (int i = 2; i < C; i += 2) {
                            Q0 = fma2(U0, tab.c2[i / 2], tab.d2[i / 2]);
                            Q1 = fma2(U1, tab.c2[i / 2], tab.d2[i / 2]);
                            Th0 = fma2(Th0, pk2(ss0, ss0), mul2(Q0, ldp(rp0, i)));
                            Th1 = fma2(Th1, pk2(ss1, ss1), mul2(Q1, ldp(rp1, i)));
                        }
                        float se0, so0, te0, to0, se1, so1, te1, to1;
                        upk2(Sh0, se0, so0);
                        upk2(Th0, te0, to0);
                        upk2(Sh1, se1, so1);
                        upk2(Th1, te1, to1);
                        g0 = P00 * fmaf(s0, to0, fmaf(ss0, te0, fmaf(r0, so0, se0)));
                        g1 = P01 * fmaf(s1, to1, fmaf(ss1, te1, fmaf(r1, so1, se1)));
                    }
                }
                if (rare && lo_j >= 0) {  // exact window edges / record clipping / exact-ToF groups
#pragma unroll 1
                    for (int h = 0; h < 2; ++h) {
                        const int64_t gi = (int64_t)cb * CELL + li + h;
                        const int pb = ((li + h) >> 1) * 4 + ((li + h) & 1);
                        const float4 kdt = make_float4(s_kxy[pb], s_kxy[pb + 2], s_kzw[pb], s_kzw[pb + 2]);
                        const PairWin pw = pair_setup<SDEG>(a, kdt, 1.f, orig, gi, Mpad, sx, sy, sz, k);
                        float part = 0.f;
                        const float* rq = ADJT_DBL ? (const float*)(col2 + (pw.n_lo - lo_j) * 32) : col + (pw.n_lo - lo_j) * 32;
                        for (int m = 0; m < pw.cnt; ++m) {
                            const float um = pw.u_lo - (float)m;
                            part = fmaf(um * ex2f((um * k.K1u) * um), rq[m * 32 * (1 + ADJT_DBL)], part);
                        }
                        if (h) g1 = pw.w * part; else g0 = pw.w * part;
                    }
                }
                gv[t] = g0;
                gv[t + 1] = g1;
            }
            warp_reduce_scatter8(gv, lane, s_g + warp * (STAGE_CELLS * CELL) + gq * GROUP);
        }
        __syncthreads();
        write_group_partials(s_g, nw, nc, gpart + (int64_t)(blockIdx.y + k.grp0) * Mpad + (int64_t)cb * CELL);
    }
}

// ------------------------------------------------------------------ adjoint, lane-centred factorisation (fp64 chains)
// k_adjoint_t's decomposition (lane = sensor, the lane's residual window in a private
// smem column, fp64 anchor per 8-kernel group) with the Gaussian factorised about the
// CENTRE of the lane's column.  Column index t, T = La / 2, G(t) = 2^{K (t - T)^2}.
// A pair's window is t_c + m, m in [-C, W - C) (t_c = o + C, C = W / 2) with
// u = u_c - m, u_c = u_lo - C in (-1, 0], and
//   (u_c - m) 2^{K (u_c - m)^2} = E Ginv(t_c) G(t_c + m) R^m (u_c - m),
//   E = 2^{K u_c^2},   R = 2^{-2K (u_c + t_c - T)} = r Q(t_c),   r = 2^{-2K u_c},
//   Q(t) = 2^{-2K (t - T)},  Ginv = 1 / G.
// The column is staged once per region as dtil_t = delta_t G(t) (fp64), so
//   g_ij = w E Ginv(t_c) [u_c (U + L) - R U' + L#],
//   U = sum_{m=0}^{W-C-1} dtil_{t_c+m} R^m,  U' = dU/dR,
//   L = sum_{k=1}^{C} dtil_{t_c-k} S^k,  S = 1 / R,  L# = S dL/dS,
// two simultaneous Horner chains per half, one DFMA per chain and sample.  The chains,
// R, S, E and the weight are fp64: in fp32 the rounding of R enters every power R^m and
// made the gradient's error 2e-7 (rel L2); the fp64 pipe (64 DFMA / clk / SM)
// carries two DFMA per pair-sample plus ~30 per pair.  r, 1 / r and E are short fp64
// polynomials of |z| <= 0.3 (truncation < 4e-10); G, Ginv, Q, 1 / Q are fp64 tables
// (host exp2).  Valid while G stays a normal fp32 (GPAIR_LCF_COL32): |K| max(T, La - T)^2 <= 100.
#ifndef GPAIR_LCF_WARPS
#define GPAIR_LCF_WARPS 4
#endif
#ifndef GPAIR_LCF_MINB
#define GPAIR_LCF_MINB 4
#endif
constexpr int LCF_WARPS = GPAIR_LCF_WARPS;  // sensor warps per CTA (the fp64 column costs La * 256 B per warp)
constexpr int LCF_STAGE = 4;                // cells per staged kernel tile (4 CTAs of 4 warps per SM at La = 48)
#ifndef GPAIR_LCF_PACKS
#define GPAIR_LCF_PACKS 2
#endif
constexpr int LCF_PACKS = GPAIR_LCF_PACKS;  // f32x2 time-of-flight packs per step
constexpr int LCF_PPS = 2 * LCF_PACKS;      // pairs (kernels) per step: independent fp64 chains
#ifndef GPAIR_LCF_COL32
#define GPAIR_LCF_COL32 0
#endif
#if GPAIR_LCF_COL32
typedef float lcol_t;
#else
typedef double lcol_t;
#endif

template <int W, int SDEG>
__global__ void __launch_bounds__(32 * LCF_WARPS, GPAIR_LCF_MINB)
    k_adjoint_lcf(const float4* __restrict__ kd, const float4* __restrict__ grp, const float* __restrict__ orig,
                  const float* __restrict__ sens, const int32_t* __restrict__ wlo, const float* __restrict__ resid,
                  const double* __restrict__ gtab, gacc_t* __restrict__ gpart, int32_t cpr, int32_t ncells,
                  int32_t La, int64_t Mpad, OpConst k, double Kln2) {
    constexpr int C = W / 2;
    extern __shared__ double smem8[];
    const int nw = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    gacc_t* s_g = (gacc_t*)smem8;                           // [nw][LCF_STAGE*CELL] per-warp kernel sums
    // this lane's column dtil_t = delta_t G(t) at col[t*32] (lcol_t: fp64, or fp32 widened by F2F
    // per sample -- half the shared-memory bytes, but F2F issues on the 16 / clk / SM XU pipe)
    lcol_t* col = (lcol_t*)(s_g + nw * LCF_STAGE * CELL) + (size_t)warp * La * 32 + lane;
    float4* s_grp = (float4*)((lcol_t*)(s_g + nw * LCF_STAGE * CELL) + (size_t)nw * La * 32);  // [LCF_STAGE*GPC]
    // kernel pairs interleaved: s_kxy[p] = (x0, x1, y0, y1), s_kzw[p] = (z0, z1, w0, w1)
    float* s_kxy = (float*)(s_grp + LCF_STAGE * GPC);
    float* s_kzw = s_kxy + LCF_STAGE * CELL * 2;
    double* s_gi = (double*)(s_kzw + LCF_STAGE * CELL * 2);  // [La] Ginv(t) (fp64 factor of the per-pair scale)
    for (int t = threadIdx.x; t < La; t += blockDim.x) s_gi[t] = gtab[4 * t + 2];

    const int c0 = blockIdx.x * cpr, c1 = min(c0 + cpr, ncells);
    if (c0 < c1) stage_kernel_tile(kd, grp, c0, min(LCF_STAGE, c1 - c0), s_kxy, s_kzw, s_grp);

    const int region = blockIdx.x;
    const int j = ((blockIdx.y + k.grp0) * nw + warp) * 32 + lane;
    const bool jok = j < k.Nd;
    const int lo_j = jok ? wlo[(int64_t)region * k.Nd + j] : -1;
    float sx = 0.f, sy = 0.f, sz = 0.f;
    if (jok) {
        sx = sens[j];
        sy = sens[k.Nd + j];
        sz = sens[2 * k.Nd + j];
    }
    {
        const float* src = resid + (int64_t)j * k.Nt;
        for (int t = 0; t < La; ++t) {
            const int n = lo_j + t;
            col[t * 32] = (lo_j >= 0 && n < k.Nt) ? (lcol_t)((double)src[n] * __ldg(gtab + 4 * t + 3)) : (lcol_t)0;
        }
    }
    const f2_t clo = pk2(k.c_lo, k.c_lo), mag = pk2(RND_MAGIC, RND_MAGIC), nmag = pk2(-RND_MAGIC, -RND_MAGIC);
    const f2_t one = pk2(1.f, 1.f);
    const unsigned span = (unsigned)(k.Nt - k.cnt_int);
    const double K64 = Kln2 * 1.4426950408889634;  // K of 2^{K u^2} (log2 base)
    for (int cb = c0; cb < c1; cb += LCF_STAGE) {
        const int nc = min(LCF_STAGE, c1 - cb);
        if (cb != c0) {  // the first tile was staged with the residual columns
            __syncthreads();  // every warp is done with the previous tile and its s_g sums
            stage_kernel_tile(kd, grp, cb, nc, s_kxy, s_kzw, s_grp);
        }
        __syncthreads();
        for (int gq = 0; gq < nc * GPC; ++gq) {
            const Anchor a = make_anchor(s_grp[gq], sx, sy, sz, k);
            double gv[GROUP];
            const bool exact_grp = __any_sync(0xffffffffu, a.na == NA_EXACT);
            const f2_t Ux = pk2(a.Ux, a.Ux), Uy = pk2(a.Uy, a.Uy), Uz = pk2(a.Uz, a.Uz);
            const f2_t iR2 = pk2(a.invR2, a.invR2), i2Rh = pk2(a.inv2Rh, a.inv2Rh), Eu = pk2(a.Eu, a.Eu);
            const int nrel = a.na - (RND_MAGIC_BITS - 1) - lo_j;  // o = n_lo - lo_j = bits(tt) + nrel
            // R = 2^{-2K a} with a = u_c + t_c - T = eu + cg (cg = n_a - lo_j - T, an integer per
            // group and lane): R = Ag 2^{-2K eu}, S = 1/R = Agi 2^{2K eu}; Ag, Agi once per group
            // (no per-pair table reads: shared memory is the LCF kernel's binding pipe)
            const double cgd = (double)(a.na - lo_j - (La >> 1));
            double Ag, Agi;
            exp2_pm64(-2.0 * K64 * cgd, Ag, Agi);
            // LCF_PPS kernels per step: LCF_PACKS f32x2 packs for the (fp32) time of flight
#pragma unroll
            for (int t = 0; t < GROUP; t += LCF_PPS) {
                const int li = gq * GROUP + t;
                bool rare = exact_grp;
                f2_t ulo[LCF_PACKS], twm1[LCF_PACKS], eup[LCF_PACKS];
                int o[LCF_PPS];
                if (!exact_grp) {
#pragma unroll
                    for (int h = 0; h < LCF_PACKS; ++h) {
                        const float4 pxy = *(const float4*)(s_kxy + 2 * (li + 2 * h));
                        const float4 pzw = *(const float4*)(s_kzw + 2 * (li + 2 * h));
                        const f2_t kx = pk2(pxy.x, pxy.y), ky = pk2(pxy.z, pxy.w);
                        const f2_t kz = pk2(pzw.x, pzw.y), kw = pk2(pzw.z, pzw.w);
                        const f2_t q = fma2(Ux, kx, fma2(Uy, ky, fma2(Uz, kz, kw)));
                        const f2_t eps = mul2(q, iR2);
                        f2_t S, Tw;
                        series2<SDEG>(eps, S, Tw);
                        twm1[h] = sub2(Tw, one);  // T(eps) - 1, exact (Sterbenz): w = h / 2R (1 + twm1)
                        const f2_t eu = fma2(mul2(q, i2Rh), S, Eu);
                        eup[h] = eu;
                        const f2_t x = add2(eu, clo);
                        const f2_t tt = add2(x, mag);
                        const f2_t fl = add2(tt, nmag);
                        const f2_t d = sub2(x, fl);
                        ulo[h] = sub2(eu, add2(fl, one));
                        float d0, d1, t0, t1;
                        upk2(d, d0, d1);
                        upk2(tt, t0, t1);
                        o[2 * h] = __float_as_int(t0) + nrel;
                        o[2 * h + 1] = __float_as_int(t1) + nrel;
                        rare = rare || fabsf(d0) > 0.5f - GAMMA || (unsigned)(o[2 * h] + lo_j) > span ||
                               fabsf(d1) > 0.5f - GAMMA || (unsigned)(o[2 * h + 1] + lo_j) > span;
                    }
                }
                if (!rare && lo_j >= 0) {
                    double U[LCF_PPS], Ud[LCF_PPS], Lc[LCF_PPS], Ld[LCF_PPS], R[LCF_PPS], S[LCF_PPS], uc[LCF_PPS];
                    const lcol_t* rp[LCF_PPS];
#pragma unroll
                    for (int h = 0; h < LCF_PPS; ++h) {
                        float u32a, u32b;
                        upk2(ulo[h >> 1], u32a, u32b);
                        // w E in fp32 with few roundings (the forward's scale arithmetic): its ~1 ulp
                        // per pair is below the time of flight's share of g's error
                        float sc32a, sc32b;
                        {
                            const f2_t ucp = add2(ulo[h >> 1], pk2(-(float)C, -(float)C));
                            const f2_t z = mul2(mul2(ucp, ucp), pk2((float)Kln2, (float)Kln2));
                            f2_t ep = fma2(z, pk2(1.f / 120.f, 1.f / 120.f), pk2(1.f / 24.f, 1.f / 24.f));
                            ep = fma2(z, ep, pk2(1.f / 6.f, 1.f / 6.f));
                            ep = fma2(z, ep, pk2(0.5f, 0.5f));
                            ep = fma2(z, ep, pk2(1.f, 1.f));
                            ep = fma2(z, ep, pk2(1.f, 1.f));
                            const f2_t h2 = pk2(a.h2R, a.h2R);
                            upk2(mul2(ep, fma2(h2, twm1[h >> 1], h2)), sc32a, sc32b);
                        }
                        uc[h] = (double)((h & 1) ? u32b : u32a) - (double)C;  // exact
                        const int tc = o[h] + C;
                        float e32a, e32b;
                        upk2(eup[h >> 1], e32a, e32b);
                        double ep, em;
                        exp2_pm64(-2.0 * K64 * (double)((h & 1) ? e32b : e32a), ep, em);  // 2^{-2K eu}, 2^{2K eu}
                        R[h] = Ag * ep;
                        S[h] = Agi * em;
                        rp[h] = col + tc * 32;
                        U[h] = (double)rp[h][(W - C - 1) * 32];
                        Ud[h] = 0.0;
                        Lc[h] = (double)rp[h][-C * 32];
                        Ld[h] = 0.0;
                        // scale w E Ginv(t_c), E = e^{K ln2 u_c^2}
                        gv[t + h] = (double)((h & 1) ? sc32b : sc32a) * s_gi[tc];
                    }
#pragma unroll
                    for (int i = 1; i < C; ++i) {
#pragma unroll
                        for (int h = 0; h < LCF_PPS; ++h) {
                            const int mu = W - C - 1 - i;  // upper: m = W-C-2 .. 0
                            Ud[h] = fma(Ud[h], R[h], U[h]);
                            U[h] = fma(U[h], R[h], (double)rp[h][mu * 32]);
                            const int ml = -C + i;  // lower: m = -C+1 .. -1
                            Ld[h] = fma(Ld[h], S[h], Lc[h]);
                            Lc[h] = fma(Lc[h], S[h], (double)rp[h][ml * 32]);
                        }
                    }
#pragma unroll
                    for (int i = C; i < W - C; ++i) {  // upper chain longer than the lower one (never for W % 4 == 0)
#pragma unroll
                        for (int h = 0; h < LCF_PPS; ++h) {
                            const int mu = W - C - 1 - i;
                            Ud[h] = fma(Ud[h], R[h], U[h]);
                            U[h] = fma(U[h], R[h], (double)rp[h][mu * 32]);
                        }
                    }
#pragma unroll
                    for (int h = 0; h < LCF_PPS; ++h) {
                        // L = S Lc, L# = S Lc + S^2 Ld;  u_c (U + L) - R U' + L#
                        const double Lv = S[h] * Lc[h];
                        const double Ls = fma(S[h] * S[h], Ld[h], Lv);
                        gv[t + h] *= fma(uc[h], U[h] + Lv, -R[h] * Ud[h]) + Ls;
                    }
                } else {
#pragma unroll 1
                    for (int h = 0; h < LCF_PPS; ++h) {  // exact window edges / record clipping / exact-ToF groups
                        double g = 0.0;
                        if (lo_j >= 0) {
                            const int64_t gi = (int64_t)cb * CELL + li + h;
                            const int pb = ((li + h) >> 1) * 4 + ((li + h) & 1);
                            const float4 kdt = make_float4(s_kxy[pb], s_kxy[pb + 2], s_kzw[pb], s_kzw[pb + 2]);
                            const PairWin pw = pair_setup<SDEG>(a, kdt, 1.f, orig, gi, Mpad, sx, sy, sz, k);
                            // the exact window [n_lo, n_lo + cnt) from its start t0 = n_lo - lo_j:
                            // (u - m) 2^{K (u - m)^2} = 2^{K u^2} Ginv(t0) G(t0 + m) R0^m (u - m),
                            // R0 = 2^{-2K (u + t0 - T)}: one fp64 Horner pair over the column
                            const int t0 = pw.n_lo - lo_j;
                            if (pw.cnt > 0) {
                                const double u = (double)pw.u_lo;
                                const double R0 = exp2_64(-2.0 * K64 * (u + (double)(t0 - (La >> 1))));
                                double P = col[(t0 + pw.cnt - 1) * 32], Pd = 0.0;
                                for (int m = pw.cnt - 2; m >= 0; --m) {
                                    Pd = fma(Pd, R0, P);
                                    P = fma(P, R0, (double)col[(t0 + m) * 32]);
                                }
                                g = (double)pw.w * exp2_64(K64 * u * u) * s_gi[t0] * fma(u, P, -R0 * Pd);
                            }
                        }
#pragma unroll
                        for (int hh = 0; hh < LCF_PPS; ++hh)  // static register index (h is a rolled loop)
                            if (hh == h) gv[t + hh] = g;
                    }
                }
            }
            warp_reduce_scatter8(gv, lane, s_g + warp * (LCF_STAGE * CELL) + gq * GROUP);
        }
        __syncthreads();
        write_group_partials(s_g, nw, nc, gpart + (int64_t)(blockIdx.y + k.grp0) * Mpad + (int64_t)cb * CELL,
                             LCF_STAGE * CELL);
    }
}

// ------------------------------------------------------------------ adjoint, sensor lanes, per-sample exponential
// k_adjoint_lcf's decomposition (lane = sensor, residual column per lane, fp64
// anchor per group in registers, two kernels per f32x2 setup, warp
// reduce-scatter, per-sensor-group partials) with one MUFU.EX2 per sample: the
// fast adjoint for exact-integer windows outside the LCF range (W = 5 of cfg4',
// W > 32 of the desk workload, or |K| (La/2)^2 > LCF_KMAX).
template <int W, int SDEG>
__global__ void __launch_bounds__(256, 3) k_adjoint_sl(const float4* __restrict__ kd, const float4* __restrict__ grp,
                                                       const float* __restrict__ orig, const float* __restrict__ sens,
                                                       const int32_t* __restrict__ wlo, const float* __restrict__ resid,
                                                       gacc_t* __restrict__ gpart,
                                                       int32_t cpr, int32_t ncells, int32_t La, int64_t Mpad, OpConst k,
                                                       float K) {
    const float m2K = -2.f * K;
    extern __shared__ float4 smem4[];
    // kernel pairs interleaved: s_kxy[p] = (x0, x1, y0, y1), s_kzw[p] = (z0, z1, w0, w1)
    float* s_kxy = (float*)smem4;
    float* s_kzw = s_kxy + STAGE_CELLS * CELL * 2;
    float4* s_grp = (float4*)(s_kzw + STAGE_CELLS * CELL * 2);  // [STAGE_CELLS*GPC]
    const int nw = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    gacc_t* s_g = (gacc_t*)(s_grp + STAGE_CELLS * GPC);  // [nw][STAGE_CELLS*CELL] per-warp kernel sums
    float* col = (float*)(s_g + nw * STAGE_CELLS * CELL) + (size_t)warp * La * 32 + lane;  // this lane's column delta_t
    const int region = blockIdx.x;
    const int c0 = region * cpr, c1 = min(c0 + cpr, ncells);
    if (c0 < c1) stage_kernel_tile(kd, grp, c0, min(STAGE_CELLS, c1 - c0), s_kxy, s_kzw, s_grp);
    const int j = ((blockIdx.y + k.grp0) * nw + warp) * 32 + lane;
    const bool jok = j < k.Nd;
    const int lo_j = jok ? wlo[(int64_t)region * k.Nd + j] : -1;
    float sx = 0.f, sy = 0.f, sz = 0.f;
    if (jok) {
        sx = sens[j];
        sy = sens[k.Nd + j];
        sz = sens[2 * k.Nd + j];
    }
    {
        const float* src = resid + (int64_t)j * k.Nt;
        for (int t = 0; t < La; ++t) {
            const int n = lo_j + t;
            col[t * 32] = (lo_j >= 0 && n < k.Nt) ? src[n] : 0.f;
        }
    }
    const int Tc = La >> 1;
    const f2_t c8 = pk2(1.f / 8.f, 1.f / 8.f), c4 = pk2(-0.25f, -0.25f), one = pk2(1.f, 1.f);
    const f2_t c38 = pk2(3.f / 8.f, 3.f / 8.f), c2 = pk2(-0.5f, -0.5f);
    const f2_t clo = pk2(k.c_lo, k.c_lo), mag = pk2(RND_MAGIC, RND_MAGIC), nmag = pk2(-RND_MAGIC, -RND_MAGIC);
    const f2_t K2 = pk2(K, K), M2K = pk2(m2K, m2K);
    const unsigned span = (unsigned)(k.Nt - k.cnt_int);
    for (int cb = c0; cb < c1; cb += STAGE_CELLS) {
        const int nc = min(STAGE_CELLS, c1 - cb);
        if (cb != c0) {  // the first tile was staged with the residual columns
            __syncthreads();  // every warp is done with the previous tile and its s_g sums
            stage_kernel_tile(kd, grp, cb, nc, s_kxy, s_kzw, s_grp);
        }
        __syncthreads();
        for (int gq = 0; gq < nc * GPC; ++gq) {
            const Anchor a = make_anchor(s_grp[gq], sx, sy, sz, k);
            float gv[GROUP];
            const bool exact_grp = __any_sync(0xffffffffu, a.na == NA_EXACT);
            const f2_t Ux = pk2(a.Ux, a.Ux), Uy = pk2(a.Uy, a.Uy), Uz = pk2(a.Uz, a.Uz);
            const f2_t iR2 = pk2(a.invR2, a.invR2), i2Rh = pk2(a.inv2Rh, a.inv2Rh);
            const f2_t Eu = pk2(a.Eu, a.Eu), h2R = pk2(a.h2R, a.h2R);
            const int nrel = a.na - (RND_MAGIC_BITS - 1) - lo_j;  // o = n_lo - lo_j = bits(tt) + nrel
            const float cg = (float)(a.na - lo_j - Tc);            // a_pair = eu + cg (exact integer shift)
            const f2_t CG = pk2(cg, cg);
            // four kernels per step: two f32x2 packs whose Horner chains interleave (ILP)
#pragma unroll
            for (int t = 0; t < GROUP; t += 4) {
                const int li = gq * GROUP + t;
                bool rare = exact_grp;
                f2_t eu[2], w[2], ulo[2];
                int o[4];
                if (!exact_grp) {
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const float4 pxy = *(const float4*)(s_kxy + 2 * (li + 2 * h));
                        const float4 pzw = *(const float4*)(s_kzw + 2 * (li + 2 * h));
                        const f2_t kx = pk2(pxy.x, pxy.y), ky = pk2(pxy.z, pxy.w);
                        const f2_t kz = pk2(pzw.x, pzw.y), kw = pk2(pzw.z, pzw.w);
                        const f2_t q = fma2(Ux, kx, fma2(Uy, ky, fma2(Uz, kz, kw)));
                        const f2_t eps = mul2(q, iR2);
                        f2_t S, Tw;
                        series2<SDEG>(eps, S, Tw);
                        eu[h] = fma2(mul2(q, i2Rh), S, Eu);
                        w[h] = mul2(h2R, Tw);
                        const f2_t x = add2(eu[h], clo);
                        const f2_t tt = add2(x, mag);
                        const f2_t fl = add2(tt, nmag);
                        const f2_t d = sub2(x, fl);
                        ulo[h] = sub2(eu[h], add2(fl, one));
                        float d0, d1, t0, t1;
                        upk2(d, d0, d1);
                        upk2(tt, t0, t1);
                        o[2 * h] = __float_as_int(t0) + nrel;
                        o[2 * h + 1] = __float_as_int(t1) + nrel;
                        rare = rare || fabsf(d0) > 0.5f - GAMMA || (unsigned)(o[2 * h] + lo_j) > span ||
                               fabsf(d1) > 0.5f - GAMMA || (unsigned)(o[2 * h + 1] + lo_j) > span;
                    }
                }
                if (!rare && lo_j >= 0) {
                    // one MUFU.EX2 per sample: g = w sum_m u_m 2^{K u_m^2} delta[o + m], u_m = u_lo - m
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const float* rp0 = col + o[2 * h] * 32;
                        const float* rp1 = col + o[2 * h + 1] * 32;
                        f2_t u2 = ulo[h];
                        f2_t acc2 = pk2(0.f, 0.f);
#pragma unroll
                        for (int m = 0; m < W; ++m) {
                            float a0, a1;
                            upk2(mul2(mul2(u2, K2), u2), a0, a1);
                            acc2 = fma2(mul2(u2, pk2(ex2f(a0), ex2f(a1))), pk2(rp0[m * 32], rp1[m * 32]), acc2);
                            u2 = add2(u2, pk2(-1.f, -1.f));
                        }
                        float v0, v1, w0, w1;
                        upk2(acc2, v0, v1);
                        upk2(w[h], w0, w1);
                        gv[t + 2 * h] = w0 * v0;
                        gv[t + 2 * h + 1] = w1 * v1;
                    }
                } else {
#pragma unroll
                    for (int h = 0; h < 4; ++h) {  // exact window edges / record clipping / exact-ToF groups
                        float g = 0.f;
                        if (lo_j >= 0) {
                            const int64_t gi = (int64_t)cb * CELL + li + h;
                            const int pb = ((li + h) >> 1) * 4 + ((li + h) & 1);
                            const float4 kdt = make_float4(s_kxy[pb], s_kxy[pb + 2], s_kzw[pb], s_kzw[pb + 2]);
                            const PairWin pw = pair_setup<SDEG>(a, kdt, 1.f, orig, gi, Mpad, sx, sy, sz, k);
                            float part = 0.f;
                            const int oo = pw.n_lo - lo_j;
                            for (int m = 0; m < pw.cnt; ++m) {
                                const float um = pw.u_lo - (float)m;
                                part = fmaf(um * ex2f((um * k.K1u) * um), col[(oo + m) * 32], part);
                            }
                            g = pw.w * part;
                        }
                        gv[t + h] = g;
                    }
                }
            }
            warp_reduce_scatter8(gv, lane, s_g + warp * (STAGE_CELLS * CELL) + gq * GROUP);
        }
        __syncthreads();
        write_group_partials(s_g, nw, nc, gpart + (int64_t)(blockIdx.y + k.grp0) * Mpad + (int64_t)cb * CELL);
    }
}

// sum of the sensor-group partial gradients (fixed order) + epilogue
template <int MODE>
__global__ void k_adj_gather(const gacc_t* __restrict__ gpart, int32_t ngroups, const int32_t* __restrict__ perm,
                             int64_t Mpad, EpiParams ep) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= Mpad) return;
    const int32_t ic = perm[i];
    if (ic < 0) return;
    gacc_t acc = 0;
    for (int g = 0; g < ngroups; ++g) acc += gpart[(int64_t)g * Mpad + i];
    adjoint_epilogue<MODE>((float)acc, ic, ep);
}

}  // namespace
int pick_wmax(int w) {
    static const int opts[] = {5, 8, 12, 16, 20, 24, 32, 48, 64};
    for (int o : opts)
        if (w <= o) return o;
    return 64;
}
namespace {

template <int W, int SER, bool UNION = false>
cudaError_t fwd_launch(gpair_ctx* c, cudaStream_t st) {
    constexpr bool DBUFL = (SER == 0 || SER == SER_FAST5) && W >= 12;
    size_t smem = (DBUFL ? (size_t)2 * FWD_BUF * 4
                         : (size_t)STAGE_CELLS * CELL * 20 + STAGE_CELLS * GPC * 16 +
                               (SER == SER_GEN ? (size_t)STAGE_CELLS * CELL * 16 : 0)) +
                  (size_t)c->f_warps * c->Lf * 32 * 4;
    cudaError_t e = cudaFuncSetAttribute(k_forward<W, SER, UNION>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    // lng / lg0: window of 256-sensor pipeline groups; one CTA covers 32 f_warps / f_split sensors
    const int per256 = 256 / (32 * (c->f_warps / c->f_split));
    dim3 grid(c->f_regions, c->lng > 0 ? std::min(c->lng * per256, c->f_sgroups - c->lg0 * per256) : c->f_sgroups);
    OpConst kk = c->k;
    kk.grp0 = c->lng > 0 ? c->lg0 * per256 : 0;
    ++c->n_launch;
    k_forward<W, SER, UNION><<<grid, 32 * c->f_warps, smem, st>>>(c->d_kd, c->d_amp, c->d_grp, c->d_orig, c->d_sens,
                                                      c->d_wlo_f, c->d_partial, c->f_cpr, c->ncells, c->Lf,
                                                      c->Mpad, kk, c->d_ksig, c->tab, c->f_split);
    return cudaGetLastError();
}

template <int W, int SER, int MODE>
cudaError_t adj_launch(gpair_ctx* c, const float* resid, const EpiParams& ep, cudaStream_t st) {
    size_t smem = (size_t)c->a_cpr * GPC * 33 * sizeof(Anchor) + 32 * 4 + 32 * 16 +
                  (MODE == MODE_COUNT ? 0 : (size_t)32 * c->La * 4);
    cudaError_t e = cudaFuncSetAttribute(k_adjoint<W, SER, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int threads = 32 * std::max(c->a_cpr, 1);
    ++c->n_launch;
    k_adjoint<W, SER, MODE><<<c->a_regions, threads, smem, st>>>(c->d_kd, c->d_grp, c->d_orig, c->d_perm, c->d_sens,
                                                           c->d_wlo_a, resid, c->a_cpr, c->ncells, c->La, c->Mpad,
                                                           c->k, ep, c->d_count, c->d_ksig);
    return cudaGetLastError();
}

constexpr int ADJT_WARPS = 8;  // sensor warps per CTA of k_adjoint_t

size_t adj_t_smem(const gpair_ctx* c) {
    return (size_t)STAGE_CELLS * CELL * 16 + STAGE_CELLS * GPC * 16 + (size_t)ADJT_WARPS * STAGE_CELLS * CELL * sizeof(gacc_t) +
           (size_t)ADJT_WARPS * c->La * 32 * 4 * (1 + ADJT_DBL);
}

template <int W, int MODE, int SDEG>
cudaError_t adj_t_launch(gpair_ctx* c, const float* resid, const EpiParams& ep, cudaStream_t st) {
    const int nw = ADJT_WARPS;
    const size_t smem = adj_t_smem(c);
    cudaError_t e = cudaFuncSetAttribute(k_adjoint_t<W, SDEG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int ngroups = (c->Nd + 32 * nw - 1) / (32 * nw);
    dim3 grid(c->a_regions, c->lng > 0 ? c->lng : ngroups);
    OpConst kk = c->k;
    kk.grp0 = c->lng > 0 ? c->lg0 : 0;
    ++c->n_launch;
    k_adjoint_t<W, SDEG><<<grid, 32 * nw, smem, st>>>(c->d_kd, c->d_grp, c->d_orig, c->d_sens, c->d_wlo_a, resid, c->d_gpart,
                                                c->a_cpr, c->ncells, c->La, c->Mpad, kk, c->tab);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    if (c->lskip_gather) return cudaSuccess;  // pipelined iterate: launched once after all groups
    ++c->n_launch;
    k_adj_gather<MODE><<<(unsigned)((c->Mpad + 255) / 256), 256, 0, st>>>(c->d_gpart, ngroups, c->d_perm, c->Mpad, ep);
    return cudaGetLastError();
}

size_t adj_lcf_smem(const gpair_ctx* c) {
    return (size_t)LCF_STAGE * CELL * 16 + LCF_STAGE * GPC * 16 + (size_t)LCF_WARPS * LCF_STAGE * CELL * sizeof(gacc_t) +
           (size_t)c->La * 8 + (size_t)LCF_WARPS * c->La * 32 * sizeof(lcol_t);
}

template <int W, int MODE, int SDEG>
cudaError_t adj_lcf_launch(gpair_ctx* c, const float* resid, const EpiParams& ep, cudaStream_t st) {
    const int nw = LCF_WARPS;
    const size_t smem = adj_lcf_smem(c);
    cudaError_t e = cudaFuncSetAttribute(k_adjoint_lcf<W, SDEG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int ngroups = (c->Nd + 32 * nw - 1) / (32 * nw);
    constexpr int per256 = 256 / (32 * LCF_WARPS);  // adjoint sensor groups per pipeline (256-sensor) group
    dim3 grid(c->a_regions, c->lng > 0 ? std::min(c->lng * per256, ngroups - c->lg0 * per256) : ngroups);
    OpConst kk = c->k;
    kk.grp0 = c->lng > 0 ? c->lg0 * per256 : 0;
    const double Kln2 = -0.5 * c->k.h * c->k.h / (c->k.sigma * c->k.sigma);  // K ln 2 = -h^2 / (2 sigma^2)
    ++c->n_launch;
    k_adjoint_lcf<W, SDEG><<<grid, 32 * nw, smem, st>>>(c->d_kd, c->d_grp, c->d_orig, c->d_sens, c->d_wlo_a, resid,
                                                         c->d_gtab, c->d_gpart, c->a_cpr, c->ncells, c->La, c->Mpad, kk,
                                                         Kln2);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    if (c->lskip_gather) return cudaSuccess;  // pipelined iterate: launched once after all groups
    ++c->n_launch;
    k_adj_gather<MODE><<<(unsigned)((c->Mpad + 255) / 256), 256, 0, st>>>(c->d_gpart, ngroups, c->d_perm, c->Mpad, ep);
    return cudaGetLastError();
}

size_t adj_sl_smem(const gpair_ctx* c) {
    return (size_t)STAGE_CELLS * CELL * 16 + STAGE_CELLS * GPC * 16 + (size_t)ADJT_WARPS * STAGE_CELLS * CELL * sizeof(gacc_t) +
           (size_t)ADJT_WARPS * c->La * 32 * 4;
}

template <int W, int MODE, int SDEG>
cudaError_t adj_sl_launch(gpair_ctx* c, const float* resid, const EpiParams& ep, cudaStream_t st) {
    const int nw = ADJT_WARPS;
    const size_t smem = adj_sl_smem(c);
    cudaError_t e = cudaFuncSetAttribute(k_adjoint_sl<W, SDEG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int ngroups = (c->Nd + 32 * nw - 1) / (32 * nw);
    dim3 grid(c->a_regions, c->lng > 0 ? c->lng : ngroups);
    OpConst kk = c->k;
    kk.grp0 = c->lng > 0 ? c->lg0 : 0;
    ++c->n_launch;
    k_adjoint_sl<W, SDEG><<<grid, 32 * nw, smem, st>>>(c->d_kd, c->d_grp, c->d_orig, c->d_sens, c->d_wlo_a, resid,
                                                       c->d_gpart, c->a_cpr, c->ncells, c->La, c->Mpad, kk,
                                                       c->k.K1u);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    if (c->lskip_gather) return cudaSuccess;  // pipelined iterate: launched once after all groups
    ++c->n_launch;
    k_adj_gather<MODE><<<(unsigned)((c->Mpad + 255) / 256), 256, 0, st>>>(c->d_gpart, ngroups, c->d_perm, c->Mpad, ep);
    return cudaGetLastError();
}

template <int MODE, int SDEG>
cudaError_t adj_sl_dispatch(gpair_ctx* c, const float* resid, const EpiParams& ep, cudaStream_t st) {
    switch (c->k.cnt_int) {
        case 5: return adj_sl_launch<5, MODE, SDEG>(c, resid, ep, st);
        case 8: return adj_sl_launch<8, MODE, SDEG>(c, resid, ep, st);
        case 12: return adj_sl_launch<12, MODE, SDEG>(c, resid, ep, st);
        case 16: return adj_sl_launch<16, MODE, SDEG>(c, resid, ep, st);
        case 20: return adj_sl_launch<20, MODE, SDEG>(c, resid, ep, st);
        case 24: return adj_sl_launch<24, MODE, SDEG>(c, resid, ep, st);
        case 32: return adj_sl_launch<32, MODE, SDEG>(c, resid, ep, st);
        case 48: return adj_sl_launch<48, MODE, SDEG>(c, resid, ep, st);
        default: return adj_sl_launch<64, MODE, SDEG>(c, resid, ep, st);
    }
}

template <int SER, int MODE>
cudaError_t adj_dispatch2(gpair_ctx* c, const float* resid, const EpiParams& ep, cudaStream_t st) {
    switch (pick_wmax(c->k.wmax)) {
        case 5: return adj_launch<5, SER, MODE>(c, resid, ep, st);
        case 8: return adj_launch<8, SER, MODE>(c, resid, ep, st);
        case 12: return adj_launch<12, SER, MODE>(c, resid, ep, st);
        case 16: return adj_launch<16, SER, MODE>(c, resid, ep, st);
        case 20: return adj_launch<20, SER, MODE>(c, resid, ep, st);
        case 24: return adj_launch<24, SER, MODE>(c, resid, ep, st);
        case 32: return adj_launch<32, SER, MODE>(c, resid, ep, st);
        case 48: return adj_launch<48, SER, MODE>(c, resid, ep, st);
        default: return adj_launch<64, SER, MODE>(c, resid, ep, st);
    }
}

// general operator (row f4): windows rounded up to 8 / 16 / 32 / 64 samples
int pick_wmax_gen(int w) { return w <= 8 ? 8 : w <= 16 ? 16 : w <= 32 ? 32 : 64; }

template <int MODE>
cudaError_t adj_dispatch_gen(gpair_ctx* c, const float* resid, const EpiParams& ep, cudaStream_t st) {
    switch (pick_wmax_gen(c->k.wmax)) {
        case 8: return adj_launch<8, SER_GEN, MODE>(c, resid, ep, st);
        case 16: return adj_launch<16, SER_GEN, MODE>(c, resid, ep, st);
        case 32: return adj_launch<32, SER_GEN, MODE>(c, resid, ep, st);
        default: return adj_launch<64, SER_GEN, MODE>(c, resid, ep, st);
    }
}

}  // namespace

// Which adjoint kernel a context uses (gpair_info.adj_kernel).
int adjoint_kernel(const gpair_ctx* c) {
    if (c->ser == SER_GEN) return ADJ_LANE_KERNEL;
    if (c->mp_on) return ADJ_MP;
    const bool fast = c->ser == 0 || c->ser == SER_FAST5;
    if (fast && c->tab.on && c->d_gpart) {
        if (c->d_gtab && adj_lcf_smem(c) <= 227 * 1024 && !(c->dbg & DBG_ADJ_NO_LCF)) return ADJ_LCF;
        if (adj_t_smem(c) <= 227 * 1024 && !(c->dbg & DBG_ADJ_NO_T)) return ADJ_TAB_T;
    }
    if (fast && c->d_gpart && c->k.cnt_int <= 64 && adj_sl_smem(c) <= 227 * 1024 && !(c->dbg & DBG_ADJ_NO_T))
        return ADJ_SL;
    return ADJ_LANE_KERNEL;
}

namespace {

template <int MODE>
cudaError_t adj_dispatch(gpair_ctx* c, const float* resid, const EpiParams& ep, cudaStream_t st) {
    if constexpr (MODE != MODE_COUNT) {
        if (c->ser == SER_GEN) return adj_dispatch_gen<MODE>(c, resid, ep, st);
        const bool deg5 = c->ser == SER_FAST5;
        if (adjoint_kernel(c) == ADJ_MP) return launch_mp_adjoint(c, resid, MODE, ep, st);
        if (adjoint_kernel(c) == ADJ_LCF) {
            switch (c->k.cnt_int) {
                case 12: return deg5 ? adj_lcf_launch<12, MODE, 5>(c, resid, ep, st) : adj_lcf_launch<12, MODE, 2>(c, resid, ep, st);
                case 16: return deg5 ? adj_lcf_launch<16, MODE, 5>(c, resid, ep, st) : adj_lcf_launch<16, MODE, 2>(c, resid, ep, st);
                case 20: return deg5 ? adj_lcf_launch<20, MODE, 5>(c, resid, ep, st) : adj_lcf_launch<20, MODE, 2>(c, resid, ep, st);
                case 24: return deg5 ? adj_lcf_launch<24, MODE, 5>(c, resid, ep, st) : adj_lcf_launch<24, MODE, 2>(c, resid, ep, st);
                case 32: return deg5 ? adj_lcf_launch<32, MODE, 5>(c, resid, ep, st) : adj_lcf_launch<32, MODE, 2>(c, resid, ep, st);
                default: break;
            }
        }
        if (adjoint_kernel(c) == ADJ_SL)
            return deg5 ? adj_sl_dispatch<MODE, 5>(c, resid, ep, st) : adj_sl_dispatch<MODE, 2>(c, resid, ep, st);
        if (adjoint_kernel(c) == ADJ_TAB_T) {
            switch (c->k.cnt_int) {
                case 12: return deg5 ? adj_t_launch<12, MODE, 5>(c, resid, ep, st) : adj_t_launch<12, MODE, 2>(c, resid, ep, st);
                case 16: return deg5 ? adj_t_launch<16, MODE, 5>(c, resid, ep, st) : adj_t_launch<16, MODE, 2>(c, resid, ep, st);
                case 20: return deg5 ? adj_t_launch<20, MODE, 5>(c, resid, ep, st) : adj_t_launch<20, MODE, 2>(c, resid, ep, st);
                case 24: return deg5 ? adj_t_launch<24, MODE, 5>(c, resid, ep, st) : adj_t_launch<24, MODE, 2>(c, resid, ep, st);
                case 32: return deg5 ? adj_t_launch<32, MODE, 5>(c, resid, ep, st) : adj_t_launch<32, MODE, 2>(c, resid, ep, st);
                default: break;
            }
        }
    } else {
        if (c->ser == SER_GEN) return cudaErrorNotSupported;
    }
    return c->ser == 0 ? adj_dispatch2<0, MODE>(c, resid, ep, st)
                       : (c->ser == 2 ? adj_dispatch2<2, MODE>(c, resid, ep, st) : adj_dispatch2<5, MODE>(c, resid, ep, st));
}

template <int SER>
cudaError_t fwd_dispatch(gpair_ctx* c, cudaStream_t st) {
    switch (pick_wmax(c->k.wmax)) {
        case 5: return fwd_launch<5, SER>(c, st);
        case 8: return fwd_launch<8, SER>(c, st);
        case 12: return fwd_launch<12, SER>(c, st);
        case 16:
            if constexpr (SER == 0)
                if (c->f_union) return fwd_launch<16, 0, true>(c, st);
            return fwd_launch<16, SER>(c, st);
        case 20: return fwd_launch<20, SER>(c, st);
        case 24: return fwd_launch<24, SER>(c, st);
        case 32: return fwd_launch<32, SER>(c, st);
        case 48: return fwd_launch<48, SER>(c, st);
        default: return fwd_launch<64, SER>(c, st);
    }
}

}  // namespace

cudaError_t launch_gather(gpair_ctx* c, const float* src, int npc, float eps, cudaStream_t st) {
    ++c->n_launch;
    k_gather<<<(unsigned)((c->Mpad + 255) / 256), 256, 0, st>>>(src, c->d_perm, c->Mpad, npc, eps, c->d_amp);
    return cudaGetLastError();
}

cudaError_t launch_forward(gpair_ctx* c, cudaStream_t st) {
    if (c->ser == SER_GEN) {
        switch (pick_wmax_gen(c->k.wmax)) {
            case 8: return fwd_launch<8, SER_GEN>(c, st);
            case 16: return fwd_launch<16, SER_GEN>(c, st);
            case 32: return fwd_launch<32, SER_GEN>(c, st);
            default: return fwd_launch<64, SER_GEN>(c, st);
        }
    }
    if (c->ser == SER_FAST5) return fwd_dispatch<SER_FAST5>(c, st);
    return c->ser == 0 ? fwd_dispatch<0>(c, st) : (c->ser == 2 ? fwd_dispatch<2>(c, st) : fwd_dispatch<5>(c, st));
}

cudaError_t launch_reduce(gpair_ctx* c, float* y, const float* b, float* delta, cudaStream_t st) {
    // per-warp spans: sum <= live range + RED_WARPS (Lf - 1) + RED_WARPS
    const size_t smem = (size_t)(std::max(c->jlen_max, 1) + RED_WARPS * (c->Lf + 1)) * 8;
    cudaError_t e = cudaFuncSetAttribute(k_reduce, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    OpConst kk = c->k;
    kk.j0 = c->lnj > 0 ? c->lj0 : 0;  // lnj / lj0: sensor window (pipeline)
    ++c->n_launch;
    k_reduce<<<c->lnj > 0 ? c->lnj : c->Nd, 32 * RED_WARPS, smem, st>>>(c->d_partial, c->d_rent, c->f_regions, c->Lf, kk, y, b, delta,
                                                  c->d_loss_part, c->n_near ? c->d_near_row : nullptr, c->d_ynear);
    if (b) c->n_loss_part = c->Nd;
    return cudaGetLastError();
}

cudaError_t launch_residual(gpair_ctx* c, const float* y, const float* b, float* delta, cudaStream_t st) {
    ++c->n_launch;
    k_residual<<<c->lnj > 0 ? c->lnj : c->Nd, 256, 0, st>>>(y, b, c->Nt, delta, c->d_loss_part,
                                                            c->lnj > 0 ? c->lj0 : 0);
    c->n_loss_part = c->Nd;
    return cudaGetLastError();
}

cudaError_t launch_loss(gpair_ctx* c, float* loss_out, cudaStream_t st, const double* reg_part, int32_t n_reg,
                        double lam) {
    ++c->n_launch;
    k_loss<<<1, 1024, 0, st>>>(c->d_loss_part, c->n_loss_part, 1.0 / ((double)c->Nd * (double)c->Nt), reg_part,
                               reg_part ? n_reg : 0, lam, loss_out);
    return cudaGetLastError();
}

cudaError_t launch_adjoint(gpair_ctx* c, const float* resid, int mode, const EpiParams& ep, cudaStream_t st) {
    if (mode == EPI_GRAD) return adj_dispatch<EPI_GRAD>(c, resid, ep, st);
    if (mode == EPI_NPC_ADAM) return adj_dispatch<EPI_NPC_ADAM>(c, resid, ep, st);
    return adj_dispatch<EPI_CLAMP>(c, resid, ep, st);
}

cudaError_t launch_group_gather(gpair_ctx* c, const gacc_t* gpart, int ngroups, int mode, const EpiParams& ep,
                                cudaStream_t st) {
    const unsigned nb = (unsigned)((c->Mpad + 255) / 256);
    ++c->n_launch;
    if (mode == EPI_GRAD)
        k_adj_gather<EPI_GRAD><<<nb, 256, 0, st>>>(gpart, ngroups, c->d_perm, c->Mpad, ep);
    else if (mode == EPI_NPC_ADAM)
        k_adj_gather<EPI_NPC_ADAM><<<nb, 256, 0, st>>>(gpart, ngroups, c->d_perm, c->Mpad, ep);
    else
        k_adj_gather<EPI_CLAMP><<<nb, 256, 0, st>>>(gpart, ngroups, c->d_perm, c->Mpad, ep);
    return cudaGetLastError();
}

cudaError_t launch_adjoint_gather(gpair_ctx* c, int mode, const EpiParams& ep, cudaStream_t st) {
    return launch_group_gather(c, c->d_gpart, adjoint_groups(c), mode, ep, st);
}

int adjoint_groups(const gpair_ctx* c) {
    if (adjoint_kernel(c) == ADJ_MP) return mp_groups(c);
    const int nw = adjoint_kernel(c) == ADJ_LCF ? LCF_WARPS : ADJT_WARPS;
    return (c->Nd + 32 * nw - 1) / (32 * nw);
}

cudaError_t launch_count(gpair_ctx* c, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(c->d_count, 0, sizeof(unsigned long long), st);
    if (e != cudaSuccess) return e;
    EpiParams ep{};
    return adj_dispatch<MODE_COUNT>(c, nullptr, ep, st);
}

}  // namespace gpair
