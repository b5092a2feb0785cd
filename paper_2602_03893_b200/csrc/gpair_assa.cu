// gpair_assa.cu -- the paper's ASSA operator (PAPER.md
// Eqs. 8-17 and Algorithm 1), B200-native.
//
// Forward (Eq. 13, y = S_down(h * P_up x)) in the paper's own structure, with
// the intermediate buffer kept on chip:
//   k_assa_forward  lane = sensor, warp = 32 sensors, CTA = region of cells.
//                   P_up (Eq. 9): every pair adds A_i / r_ij into its sensor's
//                   upsampled histogram z_j[k_ij] held in a private shared-
//                   memory column (one RMW per pair, no atomics); then each
//                   lane evaluates the transposed convolution (Eq. 10) only at
//                   the decimated points alpha n (Eq. 12) and the region trace
//                   is flushed like k_forward (same partial layout, reduced by
//                   k_reduce in a fixed order).
// Adjoint (Eq. 14, g = P_up^T (h-bar * S_down^T delta)):
//   k_assa_dconv    zero-fill (Eq. 15) + correlation with h-bar (Eq. 16), one
//                   thread per upsampled sample: dconv_j[q] = sum_n h[alpha n - q] delta_j[n].
//   k_assa_adjoint  lane = kernel: back-projection (Eq. 17) g_i = sum_j
//                   dconv_j[k_ij] / r_ij from dconv windows staged in shared
//                   memory, fused with the same update epilogue as k_adjoint.
// k_ij and the weight 1/r_ij come from assa_setup() (gpair_internal.cuh): the
// fp64 group anchors of the exact operator, with an fp64 re-decision of the
// rounding (bit-identical to the oracle) when alpha eu + 1/2 is near an integer.
#include <algorithm>

#include "gpair_ctx.h"

namespace gpair {

namespace {

constexpr int A_STAGE = 8;     // cells staged per step
#ifndef GPAIR_ASSA_WARPS
#define GPAIR_ASSA_WARPS 3
#endif
constexpr int A_WARPS = GPAIR_ASSA_WARPS;  // sensor warps per forward CTA
constexpr int MAX_TAPS = 1024; // 2K+1 limit of the shared-memory taps table

// Histogram column layout (per lane): ZG zero guard rows, the alpha*Lf rows of
// z, ZG zero guard rows (so the convolution needs no bounds checks), and, when
// the convolution cannot run in place, Lf output rows.  In place: output chunk
// c (CONV_CHUNK rows) is written over z rows [c C, c C + C) after it is
// computed; later chunks only read z rows >= alpha (c+1) C - K, which is past
// them iff K <= C (alpha - 1).
constexpr int CONV_CHUNK = 16;
__host__ __device__ inline int zguard(int K) { return K > 16 ? K : 16; }
// (only the chunked register path, K <= 16, writes in place; the generic path
// writes each output immediately and therefore always uses separate rows)
__host__ __device__ inline bool conv_inplace(int alpha, int K) {
    return K <= 16 && alpha >= 2 && K <= CONV_CHUNK * (alpha - 1);
}
int zrows_of(int alpha, int K, int Lf) {
    return alpha * Lf + 2 * zguard(K) + (conv_inplace(alpha, K) ? 0 : Lf);
}

template <int SER>
__global__ void __launch_bounds__(32 * A_WARPS) k_assa_forward(
    const float4* __restrict__ kd, const float* __restrict__ amp, const float4* __restrict__ grp,
    const float* __restrict__ orig, const float* __restrict__ sens, const int32_t* __restrict__ wlo,
    const float* __restrict__ taps, float* __restrict__ partial, int32_t cpr, int32_t ncells, int32_t Lf,
    int32_t zrows, int64_t Mpad, OpConst k) {
    extern __shared__ float4 smem4[];
    // kernel pairs interleaved: s_kxy[p] = (x0, x1, y0, y1), s_kzw[p] = (z0, z1, w0, w1) (f32x2 set-up)
    float* s_kxy = (float*)smem4;                        // [A_STAGE*32*2]
    float* s_kzw = s_kxy + A_STAGE * CELL * 2;           // [A_STAGE*32*2]
    float4* s_grp = smem4 + A_STAGE * CELL;              // [A_STAGE*GPC]
    float* s_amp = (float*)(s_grp + A_STAGE * GPC);      // [A_STAGE*32]
    float* s_taps = s_amp + A_STAGE * CELL;              // [2K+1] (padded to 4)
    const int ntaps = 2 * k.K + 1;
    const int nw = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float* s_z = s_taps + ((ntaps + 3) & ~3) + (size_t)warp * zrows * 32;

    for (int t = threadIdx.x; t < ntaps; t += blockDim.x) s_taps[t] = taps[t];
    const int region = blockIdx.x;
    const int jbase = (blockIdx.y * nw + warp) * 32;
    const int j = jbase + lane;
    const bool jok = j < k.Nd;
    for (int t = lane; t < zrows * 32; t += 32) s_z[t] = 0.f;
    const int lo_j = jok ? wlo[(int64_t)region * k.Nd + j] : -1;
    const int klo = k.alpha * lo_j;  // upsampled index of the column's first row
    const int kmax = k.alpha * k.Nt;
    float sx = 0.f, sy = 0.f, sz = 0.f;
    if (jok) {
        sx = sens[j];
        sy = sens[k.Nd + j];
        sz = sens[2 * k.Nd + j];
    }
    float* zc = s_z + lane;
    const int ZG = zguard(k.K);
    float* zs = zc + ZG * 32;  // z row p of this lane's column at zs[p * 32]
    // ---- 1. projection P_up (Eq. 9): one shared-memory RMW per pair
    const int c0 = region * cpr, c1 = min(c0 + cpr, ncells);
    for (int cb = c0; cb < c1; cb += A_STAGE) {
        const int nc = min(A_STAGE, c1 - cb);
        __syncthreads();
        for (int t = threadIdx.x; t < nc * CELL; t += blockDim.x) {
            const float4 v = kd[(int64_t)cb * CELL + t];
            const int pb = (t >> 1) * 4 + (t & 1);
            s_kxy[pb] = v.x;
            s_kxy[pb + 2] = v.y;
            s_kzw[pb] = v.z;
            s_kzw[pb + 2] = v.w;
            s_amp[t] = amp[(int64_t)cb * CELL + t];
        }
        if (threadIdx.x < nc * GPC) s_grp[threadIdx.x] = grp[(int64_t)cb * GPC + threadIdx.x];
        __syncthreads();
        for (int gq = 0; gq < nc * GPC && lo_j >= 0; ++gq) {
            const Anchor a = make_anchor(s_grp[gq], sx, sy, sz, k);
            const bool fast = SER <= 2 && !__any_sync(__activemask(), a.na == NA_EXACT);
            const float* ampg = s_amp + gq * GROUP;
            const int64_t gi0 = (int64_t)cb * CELL + gq * GROUP;
            if (fast) {
                // two kernels per f32x2 step (assa_pre's arithmetic, bit-identical index decisions),
                // the group's 4 steps unrolled: 8 independent set-ups, then the RMWs (ILP)
                const f2_t Ux = pk2(a.Ux, a.Ux), Uy = pk2(a.Uy, a.Uy), Uz = pk2(a.Uz, a.Uz);
                const f2_t iR2 = pk2(a.invR2, a.invR2), i2Rh = pk2(a.inv2Rh, a.inv2Rh);
                const f2_t Eu = pk2(a.Eu, a.Eu), h2R = pk2(a.h2R, a.h2R);
                const f2_t alf = pk2((float)k.alpha, (float)k.alpha), half = pk2(0.5f, 0.5f);
                const f2_t nhalf = pk2(-0.5f, -0.5f), two_h = pk2(k.two_over_h, k.two_over_h);
                const f2_t mag = pk2(RND_MAGIC, RND_MAGIC), nmag = pk2(-RND_MAGIC, -RND_MAGIC);
                const float gam = 0.5f - GAMMA * (float)k.alpha;
                const int kna = k.alpha * a.na - RND_MAGIC_BITS - klo;  // row = bits(t) + kna
                int row[GROUP];
                float wv[GROUP];
                unsigned amb = 0;
#pragma unroll
                for (int t = 0; t < GROUP; t += 2) {
                    const int li = gq * GROUP + t;
                    const float4 pxy = *(const float4*)(s_kxy + 2 * li), pzw = *(const float4*)(s_kzw + 2 * li);
                    const f2_t A2 = *(const f2_t*)(s_amp + li);
                    const f2_t q = fma2(Ux, pk2(pxy.x, pxy.y), fma2(Uy, pk2(pxy.z, pxy.w), fma2(Uz, pk2(pzw.x, pzw.y), pk2(pzw.z, pzw.w))));
                    f2_t S, Tw;
                    series2<2>(mul2(q, iR2), S, Tw);
                    const f2_t eu = fma2(mul2(q, i2Rh), S, Eu);
                    const f2_t w2 = mul2(mul2(A2, mul2(h2R, Tw)), two_h);
                    const f2_t xa = fma2(alf, eu, half);
                    const f2_t tt = add2(add2(xa, nhalf), mag);
                    const f2_t fl = add2(tt, nmag);
                    const f2_t dd = sub2(sub2(xa, fl), half);
                    float t0, t1, d0, d1;
                    upk2(tt, t0, t1);
                    upk2(dd, d0, d1);
                    upk2(w2, wv[t], wv[t + 1]);
                    row[t] = __float_as_int(t0) + kna;
                    row[t + 1] = __float_as_int(t1) + kna;
                    amb |= (fabsf(d0) > gam ? 1u : 0u) << t;
                    amb |= (fabsf(d1) > gam ? 1u : 0u) << (t + 1);
                }
                if (amb) {
#pragma unroll
                    for (int t = 0; t < GROUP; ++t)
                        if ((amb >> t) & 1u) row[t] = assa_fix(orig, gi0 + t, Mpad, sx, sy, sz, k) - klo;
                }
#pragma unroll
                for (int t = 0; t < GROUP; ++t)  // Eq. 9: the impulse exists inside the upsampled record
                    if ((unsigned)(row[t] + klo) < (unsigned)kmax) zs[row[t] * 32] += wv[t];
            } else {
                for (int t = 0; t < GROUP; ++t) {
                    const int li = gq * GROUP + t, pb = (li >> 1) * 4 + (li & 1);
                    const float4 kdt = make_float4(s_kxy[pb], s_kxy[pb + 2], s_kzw[pb], s_kzw[pb + 2]);
                    const AssaPair p = assa_setup<SER>(a, kdt, ampg[t], orig, gi0 + t, Mpad, sx, sy, sz, k);
                    if ((unsigned)p.k < (unsigned)kmax) zs[(p.k - klo) * 32] += p.w;  // impulse exists (Eq. 9)
                }
            }
        }
    }
    __syncthreads();
    // ---- 2. transposed convolution (Eq. 10) at the decimated points (Eq. 12),
    // per lane on its own column, in chunks of 32 outputs (conv_inplace():
    // later chunks never read rows already overwritten; otherwise the outputs
    // go to rows [alpha Lf, (alpha+1) Lf)).
    // The taps are odd (h[-q] = -h[q], h[0] = 0):
    //   y[n] = sum_{q=1..K} h[q] (z[alpha n - q] - z[alpha n + q]).
    const int zlim = k.alpha * Lf;
    const bool inplace = conv_inplace(k.alpha, k.K);
    float* ys = inplace ? zs : zs + (zlim + ZG) * 32;
    if (k.K <= 16) {
        float hq[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) hq[q] = (q + 1 <= k.K) ? s_taps[k.K + q + 1] : 0.f;
        for (int cc = 0; cc < Lf; cc += CONV_CHUNK) {
            float yv[CONV_CHUNK];
#pragma unroll
            for (int t = 0; t < CONV_CHUNK; ++t) {
                const float* zp = zs + k.alpha * (cc + t) * 32;
                float acc = 0.f;
#pragma unroll
                for (int q = 0; q < 16; ++q) {
                    acc = fmaf(hq[q], zp[-(q + 1) * 32], acc);
                    acc = fmaf(-hq[q], zp[(q + 1) * 32], acc);
                }
                yv[t] = acc;
            }
#pragma unroll
            for (int t = 0; t < CONV_CHUNK; ++t)
                if (cc + t < Lf) ys[(cc + t) * 32] = yv[t];
        }
    } else {  // long kernels (N_half >= 17 with alpha = 1): guards of K rows, separate output rows
        for (int n = 0; n < Lf; ++n) {
            const float* zp = zs + k.alpha * n * 32;
            float acc = 0.f;
            for (int q = 1; q <= k.K; ++q) {
                acc = fmaf(s_taps[k.K + q], zp[-q * 32], acc);
                acc = fmaf(-s_taps[k.K + q], zp[q * 32], acc);
            }
            ys[n * 32] = acc;
        }
    }
    __syncwarp();
    // ---- 3. flush the region trace (same layout and transpose as k_forward)
    float* s_acc = ys - lane;
    const size_t jstride = (size_t)gridDim.x * Lf;
    float* dst = partial + (size_t)jbase * jstride + (size_t)region * Lf;
    for (int m0 = 0; m0 < Lf; m0 += 32) {
        const int rows = min(32, Lf - m0);
        float v[32];
#pragma unroll
        for (int t = 0; t < 32; ++t) v[t] = (t < rows) ? s_acc[(m0 + t) * 32 + lane] : 0.f;
        __syncwarp();
#pragma unroll
        for (int t = 0; t < 32; ++t)
            if (t < rows) s_acc[(m0 + t) * 32 + (lane ^ t)] = v[t];
        __syncwarp();
        for (int jj = 0; jj < 32; ++jj)
            if (jbase + jj < k.Nd && lane < rows)
                dst[(size_t)jj * jstride + m0 + lane] = s_acc[(m0 + lane) * 32 + (jj ^ lane)];
    }
}

// zero-fill + correlation (Eqs. 15-16): dconv_j[q] = sum_{n: |alpha n - q| <= K} h[alpha n - q] delta_j[n]
__global__ void k_assa_dconv(const float* __restrict__ resid, const float* __restrict__ taps, OpConst k,
                             float* __restrict__ dconv, int64_t ld, int32_t pad, int32_t j0) {
    const int j = j0 + blockIdx.y;
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    const int Nup = k.alpha * k.Nt;
    if (q >= Nup) return;
    const float* dj = resid + (int64_t)j * k.Nt;
    const int num = q - k.K;  // n_lo = ceil((q - K) / alpha), clipped at 0
    const int nlo = max(0, num >= 0 ? (num + k.alpha - 1) / k.alpha : -((-num) / k.alpha));
    const int nhi = min(k.Nt - 1, (q + k.K) / k.alpha);
    float acc = 0.f;
    for (int n = nlo; n <= nhi; ++n) acc = fmaf(taps[k.alpha * n - q + k.K], dj[n], acc);
    dconv[(int64_t)j * ld + pad + q] = acc;
}

constexpr int MODE_COUNT = 3;

template <int SER, int MODE>
__global__ void __launch_bounds__(256) k_assa_adjoint(const float4* __restrict__ kd, const float4* __restrict__ grp,
                                                      const float* __restrict__ orig, const int32_t* __restrict__ perm,
                                                      const float* __restrict__ sens, const int32_t* __restrict__ wlo,
                                                      const float* __restrict__ dconv, int32_t cpr, int32_t ncells,
                                                      int32_t Lz, int64_t Mpad, OpConst k, EpiParams ep,
                                                      unsigned long long* count) {
    extern __shared__ float4 smem4[];
    Anchor* s_anc = (Anchor*)smem4;                          // [nw][GPC][33]
    const int nw = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float4* s_sen = (float4*)(s_anc + nw * GPC * 33);       // [32] batch sensor positions
    int32_t* s_wlo = (int32_t*)(s_sen + 32);                 // [32]
    float* s_dc = (float*)(s_wlo + 32);                      // [32][Lz]

    const int cid = blockIdx.x * cpr + warp;
    const bool cok = (warp < cpr) && (cid < ncells);
    const int64_t gi = (int64_t)cid * CELL + lane;
    float4 d4 = make_float4(0.f, 0.f, 0.f, 0.f);
    if (cok) d4 = kd[gi];
    const Anchor* my_anc = s_anc + (warp * GPC + lane / GROUP) * 33;
    const int Nup = k.alpha * k.Nt;
    float acc = 0.f;
    unsigned long long nimp = 0;
    const bool real = cok && perm[gi] >= 0;
    for (int jb = 0; jb < k.Nd; jb += 32) {
        const int nj = min(32, k.Nd - jb);
        __syncthreads();
        if (threadIdx.x < 32)
            s_wlo[threadIdx.x] = threadIdx.x < nj ? wlo[(int64_t)blockIdx.x * k.Nd + jb + threadIdx.x] : -1;
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
            for (int jj = warp; jj < 32; jj += nw) {
                const int lo = s_wlo[jj];
                const int qlo = k.alpha * lo;
                const float* src = dconv + (int64_t)(jb + jj) * Nup;
                float* dstr = s_dc + jj * Lz;
                for (int m = lane; m < Lz; m += 32) {
                    const int q = qlo + m;
                    dstr[m] = (lo >= 0 && q < Nup) ? src[q] : 0.f;
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
            const AssaPair p = (SER <= 2 && a.na != NA_EXACT)
                                   ? assa_fast(a, d4, 1.f, orig, gi, Mpad, sp.x, sp.y, sp.z, k)
                                   : assa_setup<SER>(a, d4, 1.f, orig, gi, Mpad, sp.x, sp.y, sp.z, k);
            const bool in = (unsigned)p.k < (unsigned)Nup;  // the impulse exists (Eq. 9)
            if (MODE == MODE_COUNT) {
                nimp += (real && in) ? 1ull : 0ull;
                continue;
            }
            const int row = min(max(p.k - k.alpha * lo, 0), Lz - 1);
            accb = fmaf(in ? p.w : 0.f, s_dc[jj * Lz + row], accb);  // Eq. 17
        }
        acc += accb;
    }
    if (!cok) return;
    if (MODE == MODE_COUNT) {
        for (int o = 16; o > 0; o >>= 1) nimp += __shfl_xor_sync(0xffffffffu, nimp, o);
        if (lane == 0) atomicAdd(count, nimp);
        return;
    }
    const int32_t ic = perm[gi];
    if (ic < 0) return;
    adjoint_epilogue<MODE>(acc, ic, ep);
}

template <int SER>
cudaError_t assa_fwd_launch(gpair_ctx* c, cudaStream_t st) {
    const size_t smem = assa_forward_smem(c, c->Lf);
    cudaError_t e = cudaFuncSetAttribute(k_assa_forward<SER>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    dim3 grid(c->f_regions, c->f_sgroups);
    ++c->n_launch;
    k_assa_forward<SER><<<grid, 32 * c->f_warps, smem, st>>>(c->d_kd, c->d_amp, c->d_grp, c->d_orig, c->d_sens,
                                                             c->d_wlo_f, c->d_taps, c->d_partial, c->f_cpr, c->ncells,
                                                             c->Lf, zrows_of(c->k.alpha, c->k.K, c->Lf), c->Mpad, c->k);
    return cudaGetLastError();
}

template <int SER, int MODE>
cudaError_t assa_adj_launch(gpair_ctx* c, const EpiParams& ep, cudaStream_t st) {
    const int Lz = c->k.alpha * c->La + 2 * c->k.alpha;
    size_t smem = (size_t)c->a_cpr * GPC * 33 * sizeof(Anchor) + 32 * 4 + 32 * 16 + (MODE == MODE_COUNT ? 0 : (size_t)32 * Lz * 4);
    cudaError_t e =
        cudaFuncSetAttribute(k_assa_adjoint<SER, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int threads = 32 * std::max(c->a_cpr, 1);
    ++c->n_launch;
    k_assa_adjoint<SER, MODE><<<c->a_regions, threads, smem, st>>>(c->d_kd, c->d_grp, c->d_orig, c->d_perm,
                                                                   c->d_sens, c->d_wlo_a, c->d_dconv, c->a_cpr,
                                                                   c->ncells, Lz, c->Mpad, c->k, ep, c->d_count);
    return cudaGetLastError();
}

template <int MODE>
cudaError_t assa_adj_dispatch(gpair_ctx* c, const EpiParams& ep, cudaStream_t st) {
    return c->series_small ? assa_adj_launch<2, MODE>(c, ep, st) : assa_adj_launch<5, MODE>(c, ep, st);
}

}  // namespace

size_t assa_forward_smem(const gpair_ctx* c, int Lf) {
    const int ntaps = 2 * c->k.K + 1;
    return (size_t)A_STAGE * CELL * 20 + A_STAGE * GPC * 16 + (size_t)((ntaps + 3) & ~3) * 4 +
           (size_t)c->f_warps * zrows_of(c->k.alpha, c->k.K, Lf) * 32 * 4;
}

cudaError_t launch_assa_forward(gpair_ctx* c, cudaStream_t st) {
    if (2 * c->k.K + 1 > MAX_TAPS) return cudaErrorInvalidValue;
    return c->series_small ? assa_fwd_launch<2>(c, st) : assa_fwd_launch<5>(c, st);
}

cudaError_t launch_assa_adjoint(gpair_ctx* c, const float* resid, int mode, const EpiParams& ep, cudaStream_t st) {
    if (c->mp_on) return launch_mp_adjoint(c, resid, mode, ep, st);  // gpair_mp.cu
    cudaError_t e = launch_assa_dconv(c, resid, c->d_dconv, (int64_t)c->k.alpha * c->Nt, 0, 0, c->Nd, st);
    if (e != cudaSuccess) return e;
    if (mode == EPI_GRAD) return assa_adj_dispatch<EPI_GRAD>(c, ep, st);
    if (mode == EPI_NPC_ADAM) return assa_adj_dispatch<EPI_NPC_ADAM>(c, ep, st);
    return assa_adj_dispatch<EPI_CLAMP>(c, ep, st);
}

cudaError_t launch_assa_dconv(gpair_ctx* c, const float* resid, float* out, int64_t ld, int pad, int j0, int nj,
                              cudaStream_t st) {
    const int Nup = c->k.alpha * c->Nt;
    dim3 g((Nup + 255) / 256, nj);
    ++c->n_launch;
    k_assa_dconv<<<g, 256, 0, st>>>(resid, c->d_taps, c->k, out, ld, pad, j0);
    return cudaGetLastError();
}

cudaError_t launch_assa_count(gpair_ctx* c, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(c->d_count, 0, sizeof(unsigned long long), st);
    if (e != cudaSuccess) return e;
    EpiParams ep{};
    return assa_adj_dispatch<MODE_COUNT>(c, ep, st);
}

}  // namespace gpair

namespace gpair {
int assa_forward_warps() { return A_WARPS; }
}  // namespace gpair
