// gpair_mp.cu -- the moment-polynomial adjoint (k_adjoint_mp; DESIGN.md sections 5, 6).
//
// The adjoint of Eq. 7 by transposition:
//   g_i = sum_j w_ij sum_n f(u_ijn) delta_j[n],   f(u) = u 2^{K1u u^2},  u = (r_ij - v t_n) / h,
// over the pair's window |u| < k sigma / h.  When the window length W = 2 k sigma / h is
// an exact integer (k.cnt_int) every pair whose window edge is not ambiguous covers exactly the
// W samples n_lo + m, m = 0..W-1, at u = u_lo - m with u_lo = xi0 + xi, xi0 = W/2 - 1/2 and
// xi in [-1/2, 1/2).  So a pair enters only through (n_lo, xi, w):
//   g_ij = w sum_m f(xi0 + xi - m) delta_j[n_lo + m].
// Each f(xi0 + xi - m) is smooth in xi on [-1/2, 1/2]; its interpolant at Chebyshev nodes,
// sum_k c_mk xi^k, matches it to < MP_TOL of max |f| (checked at create: degree 6 gives 3.8e-9 and
// degree 7 1.4e-10 at the bench constants, far below the fp32 time of flight's ~1e-7 per pair).
// Hence
//   g_ij = w sum_k xi^k M_k[j][n_lo],    M_k[j][n] = sum_m c_mk delta_j[n + m],
// with delta = 0 outside the record (reading R8: clipped windows, no masking).  k_mp_prep forms the
// moments of every (sensor, start sample) in fp64 once per residual, stored as 32-B rows (degree 6:
// M_0 fp64, M_1..M_6 fp32) or 48-B rows (degree 7: M_0..M_3 fp64, M_4..M_7 fp32); k_adjoint_mp then
// pays per pair one fp32 time of flight (two-level anchors, gpair_internal.cuh), one row of M from
// shared memory, an fp32 Horner tail and 1 (or 5) DFMA
// (32-B rows: the tail w xi T is summed in fp32 over a batch) -- against the LCF kernel's 16-sample fp64
// Horner chains and per-pair fp64 exponentials.  Ambiguous window edges (GAMMA band) and exact-ToF
// groups take the oracle-exact window (pair_setup) and a per-sample fp64 sum over the residual.
// The ASSA operator's adjoint (row f1) runs on the same kernel with 4-B rows of its dconv table.
//
// Layout: lane = kernel (a warp = one 32-kernel cell, a CTA = a region of mp_cpr cells); the CTA
// loops over its 256-sensor group in batches of MP_SB sensors.  Per batch the fp64 anchors (group,
// sensor) go to warp-private shared memory, f32x2-interleaved over sensor pairs, and each sensor's
// rows [lo_j, lo_j + L_r) of the table (lo_j: the region's lowest possible n_lo, k_mp_windows) are
// staged by one 1-D TMA copy (cp.async.bulk, completion on an mbarrier) into a ring of MP_NS
// stages; the last warp done with a stage refills it.  Each lane accumulates its kernel's sum over
// the group's sensors in fp64 and writes gpart[group][i]; k_adj_gather sums the groups in a fixed
// order and applies the update (deterministic, no atomics).
#include <algorithm>
#include <climits>
#include <cmath>
#include <vector>

#include "gpair_ctx.h"

namespace gpair {

namespace {

#ifndef GPAIR_MP_SB
#define GPAIR_MP_SB 16
#endif
constexpr int MP_SB = GPAIR_MP_SB;  // sensors per staged batch (8 or 16)
constexpr int MP_AJ = MP_SB / 8;    // anchor jobs per lane and batch (lane = 8 sensors x 4 groups)
constexpr int MP_SG = 256;         // sensors per CTA (blockIdx.y = sensor group = gpart row)
constexpr int32_t MP_EMPTY = INT_MIN;
constexpr double MP_TOL = 1e-8;    // max interpolation error / max |f| accepted at create (W >= 10 at k = 3)

// GPAIR_MP_CHECK=1 (a variant build, scripts/gpu_mp_check.sh): device-side bounds checks of every
// staged copy, table row and rare-path sample index; a violation traps (the launch fails loudly).
#ifndef GPAIR_MP_CHECK
#define GPAIR_MP_CHECK 0
#endif
#define MP_CHECK(cond)                        \
    do {                                      \
        if (GPAIR_MP_CHECK && !(cond)) __trap(); \
    } while (0)

__device__ __forceinline__ unsigned mp_saddr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mp_saddr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mp_saddr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(mp_saddr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n MP_WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra MP_WAIT_%=;\n}"
        ::"r"(mp_saddr(bar)), "r"(parity) : "memory");
}
// 1-D TMA: `bytes` contiguous bytes global -> shared, completion counted on `bar`
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(mp_saddr(dst)), "l"(src), "r"(bytes), "r"(mp_saddr(bar)) : "memory");
}

// Thread per (region, sensor): the range of staged rows over the region's groups, from the
// fp64 group anchors, e = (r / v - t0) f_s, r in [R - rad, R + rad], one row of margin each side:
//   exact operator: n_lo = floor(e - ku) + 1 (start sample of the window);
//   ASSA (row f1):  k_ij = floor(alpha e + 1/2) (upsampled index, Eq. 9).
// MP_EMPTY when no window / impulse reaches the record.
__global__ void k_mp_windows(const float4* __restrict__ grp, int32_t ncells, const float* __restrict__ sens,
                             int32_t cpr, int32_t nregions, OpConst k, int32_t assa, int32_t* wlo, int* maxlen) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= (int64_t)nregions * k.Nd) return;
    const int j = (int)(t % k.Nd);
    const int r = (int)(t / k.Nd);
    const double sx = sens[j], sy = sens[k.Nd + j], sz = sens[2 * k.Nd + j];
    const double ku = (double)k.ku;
    int lo = INT_MAX, hi = INT_MIN;
    const int c1 = min((r + 1) * cpr, ncells);
    for (int cc = r * cpr; cc < c1; ++cc) {
        for (int gq = 0; gq < GPC; ++gq) {
            const float4 G = grp[(int64_t)cc * GPC + gq];
            const double dx = (double)G.x - sx, dy = (double)G.y - sy, dz = (double)G.z - sz;
            const double R = sqrt(dx * dx + dy * dy + dz * dz), rad = G.w;
            const double elo = fma(R - rad, k.inv_h, -k.t0fs);
            const double ehi = fma(R + rad, k.inv_h, -k.t0fs);
            if (assa) {
                lo = min(lo, (int)floor(k.alpha * elo + 0.5) - 1);
                hi = max(hi, (int)floor(k.alpha * ehi + 0.5) + 1);
            } else {
                lo = min(lo, (int)floor(elo - ku));
                hi = max(hi, (int)floor(ehi - ku) + 2);
            }
        }
    }
    const int rmin = assa ? 0 : -(k.cnt_int - 1), rmax = assa ? k.alpha * k.Nt - 1 : k.Nt - 1;
    if (lo > hi || hi < rmin || lo > rmax) {
        wlo[(int64_t)r * k.Nd + j] = MP_EMPTY;
        return;
    }
    wlo[(int64_t)r * k.Nd + j] = lo;
    atomicMax(maxlen, hi - lo + 1);
}

// Moment table layout: [Nd][NtP] rows of 48 B, absolute row ra = n + (W - 1) + pad for start
// sample n: M_0..M_3 in fp64 (32 B) and M_4..M_7 in fp32 (16 B; their terms are below 1e-3 of
// the pair value for |xi| <= 1/2, so fp32 adds < 1e-10 relative).  Rows of n outside
// [-(W - 1), Nt - 1] are zero (set at create).  48-B rows are bank-conflict-free for any 8
// consecutive rows (row r starts at bank 12 r mod 32: 8 distinct 16-B slots).
constexpr int MP_ROW = 48;

// M_k[j][n] = sum_m c_mk delta_j[n + m] for n in [-(W - 1), Nt - 1], fp64 sums.  Thread per row.
// R32: 32-B rows of the degree-6 fit (M_0 fp64, M_1..M_6 fp32); else 48-B rows of the degree-7 fit.
template <bool R32>
__global__ void k_mp_prep(const float* __restrict__ resid, const double* __restrict__ coef, int32_t W, int32_t Nt,
                          int32_t NtP, int32_t pad, int32_t j0, char* __restrict__ Mt) {
    extern __shared__ double s_c[];  // [W][8]
    for (int t = threadIdx.x; t < W * 8; t += blockDim.x) s_c[t] = coef[t];
    __syncthreads();
    const int row = blockIdx.x * blockDim.x + threadIdx.x;  // n + W - 1
    if (row >= Nt + W - 1) return;
    const int j = j0 + blockIdx.y;
    const float* d = resid + (int64_t)j * Nt;
    const int n0 = row - (W - 1);
    double a[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    for (int m = 0; m < W; ++m) {
        const int n = n0 + m;
        const double dv = (n >= 0 && n < Nt) ? (double)__ldg(d + n) : 0.0;
        const double* c = s_c + 8 * m;
#pragma unroll
        for (int q = 0; q < 8; ++q) a[q] = fma(c[q], dv, a[q]);
    }
    MP_CHECK(row + pad >= 0 && row + pad < NtP);
    if (R32) {
        // the two 16-B chunks of absolute row ra swap places when bit 2 of ra is set: 8 consecutive
        // rows then cover the 8 16-B bank slots (blocks are staged from rows that are multiples of 8)
        const int ra = row + pad;
        char* o = Mt + ((int64_t)j * NtP + ra) * 32;
        const int sw = ((ra >> 2) & 1) * 16;
        *(double*)(o + sw) = a[0];
        *(float2*)(o + sw + 8) = make_float2((float)a[1], (float)a[2]);
        *(float4*)(o + (16 ^ sw)) = make_float4((float)a[3], (float)a[4], (float)a[5], (float)a[6]);
    } else {
        char* o = Mt + ((int64_t)j * NtP + row + pad) * MP_ROW;
        *(double2*)o = make_double2(a[0], a[1]);
        *(double2*)(o + 16) = make_double2(a[2], a[3]);
        *(float4*)(o + 32) = make_float4((float)a[4], (float)a[5], (float)a[6], (float)a[7]);
    }
}

// Anchors of a (group, sensor pair) in shared memory, f32x2-interleaved over the two sensors of
// a step: the fp32 part of the fp64 anchor (make_anchor) with n_a folded into the start row of
// the sensor's staged block, nrel = n_a - lo_j - (RND_MAGIC_BITS - 1) (NA_EXACT: exact path).
// [group][pair of sensors]: {Ux, Uy} {Uz, Eu} {invR2, inv2Rh} {h2R, nrel}, each (s0, s1).
constexpr int MP_ANC_GSTRIDE = (MP_SB / 2) * 4 + 1;  // float4 slots per group (+1: 4 groups on distinct banks)

// Rare pair: the oracle-exact window (pair_setup: exact edges, exact-ToF anchors, record
// clipping) and a per-sample fp64 sum over the residual row.
template <int SDEG>
__device__ __noinline__ double mp_rare(float4 G, float4 d4, const float* __restrict__ orig, int64_t gi, int64_t Mpad,
                                       const float* __restrict__ sens, int j, const float* __restrict__ resid,
                                       const OpConst k, double K64) {
    const float sx = sens[j], sy = sens[k.Nd + j], sz = sens[2 * k.Nd + j];
    const Anchor a = make_anchor(G, sx, sy, sz, k);
    const PairWin pw = pair_setup<SDEG>(a, d4, 1.f, orig, gi, Mpad, sx, sy, sz, k);
    MP_CHECK(pw.cnt <= 0 || (pw.n_lo >= 0 && pw.n_lo + pw.cnt <= k.Nt));
    const float* d = resid + (int64_t)j * k.Nt + pw.n_lo;
    double s = 0.0;
    for (int m = 0; m < pw.cnt; ++m) {
        const double u = (double)(pw.u_lo - (float)m);  // exact: integer shift of a small float
        s = fma(u * exp2_64(K64 * u * u), (double)d[m], s);
    }
    return (double)pw.w * s;
}

// Rare ASSA pair: assa_setup (exact-ToF anchors, fp64 re-decision of k_ij near a rounding
// edge, bit-identical to the oracle); the impulse exists only inside the upsampled record.
template <int SDEG>
__device__ __noinline__ double mp_rare_assa(float4 G, float4 d4, const float* __restrict__ orig, int64_t gi,
                                            int64_t Mpad, const float* __restrict__ sens, int j,
                                            const float* __restrict__ dtab, int32_t NtP, int32_t pad, const OpConst k) {
    const float sx = sens[j], sy = sens[k.Nd + j], sz = sens[2 * k.Nd + j];
    const Anchor a = make_anchor(G, sx, sy, sz, k);
    const AssaPair p = assa_setup<SDEG>(a, d4, 1.f, orig, gi, Mpad, sx, sy, sz, k);
    if ((unsigned)p.k >= (unsigned)(k.alpha * k.Nt)) return 0.0;
    return (double)(p.w * dtab[(int64_t)j * NtP + p.k + pad]);
}

#ifndef GPAIR_MP_NS
#define GPAIR_MP_NS 2
#endif
constexpr int MP_NS = GPAIR_MP_NS;  // staged batches in flight (ring of full mbarriers)

#ifndef GPAIR_MP_MINB
#define GPAIR_MP_MINB 3
#endif
#ifndef GPAIR_MP_TAILF32
#define GPAIR_MP_TAILF32 1
#endif
// 32-B rows: the fp32 tail w xi T of a pair is summed in fp32 over the batch (MP_SB pairs) and folded into
// the fp64 sum once per batch, so a pair costs one F2F + one DFMA (w M_0) instead of three + two
constexpr bool MP_TAILF32 = GPAIR_MP_TAILF32 != 0;
#ifndef GPAIR_MP_STAGE_UNROLL
#define GPAIR_MP_STAGE_UNROLL 1
#endif
// LR > 0: compile-time slot stride (rows per sensor in a staged batch, >= Lr2), so every staged row
// address is one add of an immediate; LR = 0: the runtime Lr2
template <int SDEG, bool ASSA, bool R32, int LR>
__global__ void __launch_bounds__(256, GPAIR_MP_MINB)
    k_adjoint_mp(const float4* __restrict__ kd, const float4* __restrict__ grp, const float* __restrict__ orig,
                 const float* __restrict__ sens, const int32_t* __restrict__ wlo, const char* __restrict__ Mt,
                 const float* __restrict__ resid, gacc_t* __restrict__ gpart, int32_t cpr, int32_t ncells,
                 int32_t Lr2, int32_t NtP, int32_t pad, int64_t Mpad, OpConst k, float xi0, double K64) {
    static_assert(MP_SB == 8 || MP_SB == 16, "anchor layout: lane = (sensor lane % 8 + 8 a, group lane / 8)");
    extern __shared__ double smem8[];
    const int nw = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int ROW = ASSA ? 4 : (R32 ? 32 : MP_ROW);             // bytes per staged row
    const int LRS = LR > 0 ? LR : Lr2;                              // rows per sensor slot
    const int sbytes = MP_SB * LRS * ROW;                           // bytes per staged batch
    char* s_M = (char*)smem8;                                       // [MP_NS][MP_SB][LRS] rows
    float4* s_anc = (float4*)(s_M + MP_NS * sbytes);                // [nw][GPC][MP_ANC_GSTRIDE]
    uint64_t* bar = (uint64_t*)(s_anc + nw * GPC * MP_ANC_GSTRIDE); // full[MP_NS]
    int* s_done = (int*)(bar + MP_NS);                              // [MP_NS] warps done with a stage

    const int W = k.cnt_int;
    const int cid = blockIdx.x * cpr + warp;
    const bool cok = cid < ncells;
    const int64_t gi = (int64_t)cid * CELL + lane;
    const float4 d4 = cok ? kd[gi] : make_float4(0.f, 0.f, 0.f, 0.f);
    const float4* grow = grp + (int64_t)(cok ? cid : 0) * GPC;
    const float4* my_anc = s_anc + (warp * GPC + (lane >> 3)) * MP_ANC_GSTRIDE;
    const int32_t* wrow = wlo + (int64_t)blockIdx.x * k.Nd;
    const int jg0 = (blockIdx.y + k.grp0) * MP_SG;
    const int jg1 = min(jg0 + MP_SG, k.Nd);
    const int nb = (jg1 - jg0 + MP_SB - 1) / MP_SB;
    const unsigned rowbytes = (unsigned)Lr2 * ROW;
    // first table row of a sensor's staged block (ASSA: 16-B aligned, Lr2 % 4 == 0)
    auto row0 = [&](int lo) {
        return lo == MP_EMPTY ? 0 : (ASSA ? ((lo + pad) & ~3) : R32 ? ((lo + W - 1 + pad) & ~7) : lo + W - 1 + pad);
    };

    // batch b's rows [lo_j, lo_j + Lr2) of every sensor by 1-D TMA into stage b % MP_NS
    // (an empty sensor copies zero rows of the table); issued by one thread
    auto issue = [&](int b) {
        const int jb = jg0 + b * MP_SB, nj = min(MP_SB, jg1 - jb);
        uint64_t* full = bar + (b % MP_NS);
        mbar_expect_tx(full, (unsigned)nj * rowbytes);
        char* dst = s_M + (b % MP_NS) * sbytes;
        for (int jj = 0; jj < nj; ++jj) {
            const int ra0 = row0(__ldg(wrow + jb + jj));
            MP_CHECK(jb + jj < k.Nd && ra0 >= 0 && ra0 + Lr2 <= NtP && (ra0 * ROW) % 16 == 0);
            tma_bulk_g2s(dst + jj * LRS * ROW, Mt + ((int64_t)(jb + jj) * NtP + ra0) * ROW, rowbytes, full);
        }
    };
    if (threadIdx.x == 0) {
        for (int s = 0; s < MP_NS; ++s) {
            mbar_init(bar + s, 1);
            s_done[s] = 0;
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0)
        for (int b = 0; b < min(MP_NS, nb); ++b) issue(b);

    const f2_t kx = pk2(d4.x, d4.x), ky = pk2(d4.y, d4.y), kz = pk2(d4.z, d4.z), kw = pk2(d4.w, d4.w);
    const f2_t clo = pk2(k.c_lo, k.c_lo), mag = pk2(RND_MAGIC, RND_MAGIC), nmag = pk2(-RND_MAGIC, -RND_MAGIC);
    const f2_t c1x = pk2(1.f + xi0, 1.f + xi0);
    const f2_t alf = pk2((float)k.alpha, (float)k.alpha), half = pk2(0.5f, 0.5f), nhalf = pk2(-0.5f, -0.5f);
    const f2_t two_h = pk2(k.two_over_h, k.two_over_h);
    const float gam_a = 0.5f - GAMMA * (float)k.alpha;
    float accf = 0.f;  // per-batch fp32 sum (ASSA: the pair values; 32-B rows: the tails), folded into acc
    // this lane's anchor job: sensor jj = lane % 8 of the batch, group gq = lane / 8 of the cell
    // (MP_SB = 16: a second job for sensor ajj + 8, 16 float4 slots further)
    const int ajj = lane & 7, agq = lane >> 3;
    float* aslot = (float*)(s_anc + (warp * GPC + agq) * MP_ANC_GSTRIDE + (ajj >> 1) * 4) + (ajj & 1);
    int lo_n[MP_AJ];  // prefetched window starts of the next batch's anchor jobs
    float sxn[MP_AJ] = {}, syn[MP_AJ] = {}, szn[MP_AJ] = {};
    auto prefetch = [&](int b) {
#pragma unroll
        for (int a = 0; a < MP_AJ; ++a) {
            const int j = jg0 + b * MP_SB + ajj + 8 * a;
            lo_n[a] = MP_EMPTY;
            if (b < nb && j < jg1) {
                lo_n[a] = __ldg(wrow + j);
                sxn[a] = __ldg(sens + j);
                syn[a] = __ldg(sens + k.Nd + j);
                szn[a] = __ldg(sens + 2 * k.Nd + j);
            }
        }
    };
    prefetch(0);
    const float4 Gq = __ldg(grow + agq);
    double acc = 0.0;
    // the ring is walked MP_NS batches at a time; ASSA unrolls it so the stage index s is a
    // compile-time constant (staged-row addresses = register + immediate; one-box A/B 15.24 -> 14.98 ms);
    // the exact operator's larger body spills when unrolled (19.8 -> 23.3 ms, variants_unroll.txt)
    constexpr int STAGE_UNROLL = (ASSA && GPAIR_MP_STAGE_UNROLL) ? MP_NS : 1;
    for (int b0 = 0; b0 < nb; b0 += MP_NS) {
#pragma unroll STAGE_UNROLL
        for (int s = 0; s < MP_NS; ++s) {
            const int b = b0 + s;
            if (b >= nb) break;
            const int jb = jg0 + b * MP_SB;
            const unsigned ph = (unsigned)(b0 / MP_NS) & 1u;
            __syncwarp();  // the previous batch's anchors are consumed
            unsigned live = 0;
#pragma unroll
            for (int aj = 0; aj < MP_AJ; ++aj) {
                const int lo_l = lo_n[aj];
                if (cok && lo_l != MP_EMPTY) {
                    const Anchor a = make_anchor(Gq, sxn[aj], syn[aj], szn[aj], k);
                    // staged row = nrel + bits(t): n_lo - lo_j (exact) or k_ij - q0 (ASSA, q0 = first staged index)
                    const int nrel = ASSA ? k.alpha * a.na - RND_MAGIC_BITS - (row0(lo_l) - pad)
                                          : a.na - (row0(lo_l) - (W - 1) - pad) - (RND_MAGIC_BITS - 1);
                    float* as = aslot + 64 * aj;
                    as[0] = a.Ux;
                    as[2] = a.Uy;
                    as[4] = a.Uz;
                    as[6] = a.Eu;
                    as[8] = a.invR2;
                    as[10] = a.inv2Rh;
                    as[12] = a.h2R;
                    as[14] = __int_as_float(a.na == NA_EXACT ? NA_EXACT : nrel);
                }
                live |= (__ballot_sync(0xffffffffu, lo_l != MP_EMPTY) & 0xFFu) << (8 * aj);
            }
            prefetch(b + 1);
            __syncwarp();
            mbar_wait(bar + s, ph);
            if (cok) {
                const char* stage = s_M + s * sbytes;
                unsigned rmask = 0;
                // one step: the pairs (kernel, sensor 2p) and (kernel, sensor 2p + 1); lv = their live bits
                auto step = [&](const int p, const unsigned lv) {
                    const float4 A0 = my_anc[4 * p], A1 = my_anc[4 * p + 1], A2 = my_anc[4 * p + 2], A3 = my_anc[4 * p + 3];
                    // fp32 time of flight of the pairs (kernel, sensor 2p) and (kernel, sensor 2p + 1) in f32x2
                    const f2_t q = fma2(pk2(A0.x, A0.y), kx, fma2(pk2(A0.z, A0.w), ky, fma2(pk2(A1.x, A1.y), kz, kw)));
                    const f2_t eps = mul2(q, pk2(A2.x, A2.y));
                    f2_t S, Tw;
                    series2<SDEG>(eps, S, Tw);
                    const f2_t eu = fma2(mul2(q, pk2(A2.z, A2.w)), S, pk2(A1.z, A1.w));
                    if constexpr (ASSA) {
                        // k_ij = alpha n_a + floor(alpha eu + 1/2), w = A / r (assa_pre's arithmetic, A = 1)
                        const f2_t w2 = mul2(mul2(pk2(A3.x, A3.y), Tw), two_h);
                        const f2_t xa = fma2(alf, eu, half);
                        const f2_t t = add2(add2(xa, nhalf), mag);
                        const f2_t fl = add2(t, nmag);
                        const f2_t dd = sub2(sub2(xa, fl), half);
                        float t0, t1, d0, d1, wa, wb;
                        upk2(t, t0, t1);
                        upk2(dd, d0, d1);
                        upk2(w2, wa, wb);
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            if (!((lv >> h) & 1u)) continue;  // warp-uniform
                            const int row = (int)((unsigned)__float_as_int(h ? A3.w : A3.z) + (unsigned)__float_as_int(h ? t1 : t0));
                            const bool rare = fabsf(h ? d1 : d0) > gam_a || (unsigned)row >= (unsigned)Lr2;
                            rmask |= (unsigned)rare << (2 * p + h);
                            const float dv = *(const float*)(stage + ((2 * p + h) * LRS + min((unsigned)row, (unsigned)Lr2 - 1u)) * 4);
                            accf = fmaf(rare ? 0.f : (h ? wb : wa), dv, accf);  // Eq. 17
                        }
                    } else {
                    const f2_t w2 = mul2(pk2(A3.x, A3.y), Tw);
                    const f2_t x = add2(eu, clo);  // alpha - 1/2, alpha = eu - ku
                    const f2_t t = add2(x, mag);
                    const f2_t fl = add2(t, nmag);  // floor(alpha) unless ambiguous
                    const f2_t dd = sub2(x, fl);    // frac(alpha) - 1/2
                    const f2_t xi2 = sub2(eu, add2(fl, c1x));  // u_lo - xi0 (exact)
                    float t0, t1, d0, d1, xa, xb, wa, wb;
                    upk2(t, t0, t1);
                    upk2(dd, d0, d1);
                    upk2(xi2, xa, xb);
                    upk2(w2, wa, wb);
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        if (!((lv >> h) & 1u)) continue;  // warp-uniform
                        const int row = (int)((unsigned)__float_as_int(h ? A3.w : A3.z) + (unsigned)__float_as_int(h ? t1 : t0));
                        const bool rare = fabsf(h ? d1 : d0) > 0.5f - GAMMA || (unsigned)row >= (unsigned)Lr2;
                        rmask |= (unsigned)rare << (2 * p + h);
                        const float xi = h ? xb : xa;
                        const float w = rare ? 0.f : (h ? wb : wa);
                        const char* rp = stage + ((2 * p + h) * LRS + min((unsigned)row, (unsigned)Lr2 - 1u)) * ROW;
                        if (R32) {  // M_0 fp64, M_1..M_6 fp32: the fp32 tail's terms are < 1/3 of the value
                            const int sw = ((int)min((unsigned)row, (unsigned)Lr2 - 1u) >> 2 & 1) * 16;
                            const float4 q0 = *(const float4*)(rp + sw);         // (M_0 lo, M_0 hi, M_1, M_2)
                            const float4 q1 = *(const float4*)(rp + (16 ^ sw));  // M_3..M_6
                            float tl = fmaf(fmaf(fmaf(q1.w, xi, q1.z), xi, q1.y), xi, q1.x);
                            tl = fmaf(fmaf(tl, xi, q0.w), xi, q0.z);
                            const double m0 = __hiloint2double(__float_as_int(q0.y), __float_as_int(q0.x));
                            if (MP_TAILF32) {
                                acc = fma((double)w, m0, acc);
                                accf = fmaf(w * xi, tl, accf);
                            } else {
                                acc = fma((double)w, fma((double)tl, (double)xi, m0), acc);
                            }
                        } else {
                            const double2 m01 = *(const double2*)rp;
                            const double2 m23 = *(const double2*)(rp + 16);
                            const float4 m47 = *(const float4*)(rp + 32);
                            const float tl = fmaf(fmaf(fmaf(m47.w, xi, m47.z), xi, m47.y), xi, m47.x);
                            const double X = (double)xi;
                            double pv = fma((double)tl, X, m23.y);
                            pv = fma(pv, X, m23.x);
                            pv = fma(pv, X, m01.y);
                            pv = fma(pv, X, m01.x);
                            acc = fma((double)w, pv, acc);
                        }
                    }
                    }
                };
                if (live == (1u << MP_SB) - 1u) {  // every sensor of the batch has a window here (common)
#pragma unroll
                    for (int p = 0; p < MP_SB / 2; ++p) step(p, 3u);
                } else {
#pragma unroll
                    for (int p = 0; p < MP_SB / 2; ++p) {
                        const unsigned lv = (live >> (2 * p)) & 3u;
                        if (lv) step(p, lv);  // warp-uniform
                    }
                }
                if (ASSA || (R32 && MP_TAILF32)) {
                    acc += (double)accf;
                    accf = 0.f;
                }
                while (rmask) {  // rare pairs of this batch (ambiguous edges / indices, exact-ToF groups)
                    const int jj = __ffs(rmask) - 1;
                    rmask &= rmask - 1u;
                    if (ASSA)
                        acc += mp_rare_assa<SDEG>(grow[lane >> 3], d4, orig, gi, Mpad, sens, jb + jj, (const float*)Mt, NtP,
                                                  pad, k);
                    else
                        acc += mp_rare<SDEG>(grow[lane >> 3], d4, orig, gi, Mpad, sens, jb + jj, resid, k, K64);
                }
            }
            // the last warp done with stage s refills it with batch b + MP_NS (no producer convoy): lane 0
            // arms the barrier, lanes 0..MP_SB-1 issue one sensor's rows each
            __syncwarp();
            int last = 0;
            if (lane == 0) {
                __threadfence_block();
                last = atomicAdd(s_done + s, 1) == nw - 1;
                if (last) s_done[s] = 0;
            }
            last = __shfl_sync(0xffffffffu, last, 0);
            if (last && b + MP_NS < nb) {
                const int jbn = jb + MP_NS * MP_SB, njn = min(MP_SB, jg1 - jbn);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                if (lane == 0) mbar_expect_tx(bar + s, (unsigned)njn * rowbytes);
                if (lane < njn) {
                    const int ra0 = row0(__ldg(wrow + jbn + lane));
                    MP_CHECK(jbn + lane < k.Nd && ra0 >= 0 && ra0 + Lr2 <= NtP && (ra0 * ROW) % 16 == 0);
                    tma_bulk_g2s(s_M + s * sbytes + lane * LRS * ROW, Mt + ((int64_t)(jbn + lane) * NtP + ra0) * ROW,
                                 rowbytes, bar + s);
                }
            }
        }
    }
    if (cok) gpart[(int64_t)(blockIdx.y + k.grp0) * Mpad + gi] = (gacc_t)acc;
}

size_t mp_smem(int Lr2, int nw, int row_bytes) {
    return (size_t)MP_NS * MP_SB * Lr2 * row_bytes + (size_t)nw * GPC * MP_ANC_GSTRIDE * 16 + MP_NS * 8 +
           MP_NS * 4;
}

// Degree-deg (<= 7) interpolation of f(xi0 + xi - m), m < W, at the deg + 1 Chebyshev nodes of
// [-1/2, 1/2] (fp64 Vandermonde solve with partial pivoting), coefficients [m][8] (zero-padded).  Returns the max error
// over a 4001-point grid relative to max |f|.
double mp_fit(int W, double K, std::vector<double>& coef, int deg) {
    constexpr int PM = 8;
    const int P = deg + 1;  // interpolation nodes / coefficients (<= 8); coef is [W][8], zero-padded
    const double xi0 = 0.5 * W - 0.5;
    double nodes[PM];
    for (int i = 0; i < P; ++i) nodes[i] = 0.5 * std::cos((2 * i + 1) * 3.141592653589793 / (2 * P));
    auto f = [&](double u) { return u * std::exp2(K * u * u); };
    coef.assign((size_t)W * PM, 0.0);
    double err = 0.0, fmax = 0.0;
    for (int m = 0; m < W; ++m) {
        double A[PM][PM + 1];
        for (int i = 0; i < P; ++i) {
            double pw = 1.0;
            for (int kk = 0; kk < P; ++kk) {
                A[i][kk] = pw;
                pw *= nodes[i];
            }
            A[i][P] = f(xi0 + nodes[i] - m);
        }
        for (int col = 0; col < P; ++col) {
            int piv = col;
            for (int r = col + 1; r < P; ++r)
                if (std::fabs(A[r][col]) > std::fabs(A[piv][col])) piv = r;
            for (int cc = 0; cc <= P; ++cc) std::swap(A[col][cc], A[piv][cc]);
            for (int r = 0; r < P; ++r) {
                if (r == col) continue;
                const double fct = A[r][col] / A[col][col];
                for (int cc = col; cc <= P; ++cc) A[r][cc] -= fct * A[col][cc];
            }
        }
        for (int kk = 0; kk < P; ++kk) coef[(size_t)m * PM + kk] = A[kk][P] / A[kk][kk];
        for (int g = 0; g <= 4000; ++g) {
            const double xi = -0.5 + g / 4000.0;
            double p = coef[(size_t)m * PM + P - 1];
            for (int kk = P - 2; kk >= 0; --kk) p = p * xi + coef[(size_t)m * PM + kk];
            const double fv = f(xi0 + xi - m);
            err = std::max(err, std::fabs(p - fv));
            fmax = std::max(fmax, std::fabs(fv));
        }
    }
    return fmax > 0.0 ? err / fmax : 1.0;
}

template <int SDEG, bool ASSA, bool R32, int LR>
cudaError_t mp_launch(gpair_ctx* c, const float* resid, int mode, const EpiParams& ep, cudaStream_t st) {
    const int G = (c->Nd + MP_SG - 1) / MP_SG;
    const int g0 = c->lng > 0 ? c->lg0 : 0;
    const int ng = c->lng > 0 ? std::min(c->lng, G - g0) : G;
    const int j0 = g0 * MP_SG, nj = std::min(c->Nd, (g0 + ng) * MP_SG) - j0;
    const int W = c->k.cnt_int;
    cudaError_t e;
    if (ASSA) {  // zero-fill + correlation (Eqs. 15-16) into the padded table
        e = launch_assa_dconv(c, resid, (float*)c->d_mp, c->mp_NtP, c->mp_pad, j0, nj, st);
    } else {
        ++c->n_launch;
        k_mp_prep<R32><<<dim3((unsigned)((c->Nt + W - 1 + 127) / 128), (unsigned)nj), 128, (size_t)W * 64, st>>>(
            resid, c->d_mp_coef, W, c->Nt, c->mp_NtP, c->mp_pad, j0, (char*)c->d_mp);
        e = cudaGetLastError();
    }
    if (e != cudaSuccess) return e;
    const size_t smem = mp_smem(LR > 0 ? LR : c->mp_Lr2, c->mp_cpr, ASSA ? 4 : c->mp_row);
    e = cudaFuncSetAttribute(k_adjoint_mp<SDEG, ASSA, R32, LR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    OpConst kk = c->k;
    kk.grp0 = g0;
    const double K64 = -1.4426950408889634 * c->k.h * c->k.h / (2.0 * c->k.sigma * c->k.sigma);
    ++c->n_launch;
    k_adjoint_mp<SDEG, ASSA, R32, LR><<<dim3((unsigned)c->mp_regions, (unsigned)ng), 32 * c->mp_cpr, smem, st>>>(
        c->d_kd, c->d_grp, c->d_orig, c->d_sens, c->d_wlo_m, (const char*)c->d_mp, resid, c->d_gpart, c->mp_cpr, c->ncells,
        c->mp_Lr2, c->mp_NtP, c->mp_pad, c->Mpad, kk, (float)(0.5 * W - 0.5), K64);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    if (c->lskip_gather) return cudaSuccess;  // pipelined iterate: launched once after all groups
    return launch_group_gather(c, c->d_gpart, G, mode, ep, st);
}

}  // namespace

int mp_groups(const gpair_ctx* c) { return (c->Nd + MP_SG - 1) / MP_SG; }

cudaError_t launch_mp_adjoint(gpair_ctx* c, const float* resid, int mode, const EpiParams& ep, cudaStream_t st) {
    if (c->assa)
        return c->series_small ? mp_launch<2, true, false, 0>(c, resid, mode, ep, st)
                               : mp_launch<5, true, false, 0>(c, resid, mode, ep, st);
    if (c->mp_row == 32) {
        const bool d2 = c->series_small != 0;
        switch (c->mp_slot) {  // compile-time slot stride (mp_setup: the smallest >= Lr2)
            case 40: return d2 ? mp_launch<2, false, true, 40>(c, resid, mode, ep, st) : mp_launch<5, false, true, 40>(c, resid, mode, ep, st);
            case 48: return d2 ? mp_launch<2, false, true, 48>(c, resid, mode, ep, st) : mp_launch<5, false, true, 48>(c, resid, mode, ep, st);
            case 64: return d2 ? mp_launch<2, false, true, 64>(c, resid, mode, ep, st) : mp_launch<5, false, true, 64>(c, resid, mode, ep, st);
            case 96: return d2 ? mp_launch<2, false, true, 96>(c, resid, mode, ep, st) : mp_launch<5, false, true, 96>(c, resid, mode, ep, st);
            default: return d2 ? mp_launch<2, false, true, 0>(c, resid, mode, ep, st) : mp_launch<5, false, true, 0>(c, resid, mode, ep, st);
        }
    }
    return c->series_small ? mp_launch<2, false, false, 0>(c, resid, mode, ep, st)
                           : mp_launch<5, false, false, 0>(c, resid, mode, ep, st);
}

// Create-time set-up: eligibility (exact-integer window on the fast anchor paths), the
// polynomial fit, the per-(region, sensor) start-sample ranges and the moment table.
cudaError_t mp_setup(gpair_ctx* c, cudaStream_t st, std::string& why) {
    c->mp_on = 0;
    const int W = c->k.cnt_int;
    const bool assa = c->assa != 0;
    if (c->gen || (c->dbg & DBG_ADJ_NO_MP)) return cudaSuccess;
    std::vector<double> coef;
    if (!assa) {
        // any exact-integer window (cnt_int > 0; not only the forward's template sizes) on the
        // anchor series paths (degree 2 when every |eps| <= EPS_SMALL, else 5 with exact-ToF groups)
        if (W < 3 || W > 128 || c->ser == SER_GEN) return cudaSuccess;
        const double K = -1.4426950408889634 * c->k.h * c->k.h / (2.0 * c->k.sigma * c->k.sigma);
        // 32-B rows (degree 6: M_0 fp64 + M_1..M_6 fp32) where that fit reaches MP_TOL, else 48-B rows
        // (degree 7: M_0..M_3 fp64 + M_4..M_7 fp32); GPAIR_MP_ROW48=1 forces the latter (A/B, tests)
        const char* r48 = std::getenv("GPAIR_MP_ROW48");
        c->mp_fit_err = mp_fit(W, K, coef, 6);
        c->mp_row = 32;
        if (!(c->mp_fit_err <= MP_TOL) || (r48 && r48[0] == '1')) {
            c->mp_fit_err = mp_fit(W, K, coef, 7);
            c->mp_row = MP_ROW;
        }
        if (!(c->mp_fit_err <= MP_TOL)) return cudaSuccess;  // short Gaussians: the LCF / sensor-lane kernels
    }
    if (!c->d_gpart) {  // contexts without the sensor-lane adjoints' group partials: allocate ours
        cudaError_t ea = cudaMalloc(&c->d_gpart, sizeof(gacc_t) * (size_t)((c->Nd + 127) / 128) * c->Mpad);
        if (ea != cudaSuccess) return ea;
        c->workspace_bytes += (int64_t)sizeof(gacc_t) * ((c->Nd + 127) / 128) * c->Mpad;
    }
    int dev_sms = 148;
    cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, c->device);
    int cpr = 8;
    if (const char* ev = std::getenv("GPAIR_MP_CPR")) cpr = std::max(1, std::min(8, atoi(ev)));  // A/B runs
    const int G = (c->Nd + MP_SG - 1) / MP_SG;
    while (cpr > 1 && (int64_t)((c->ncells + cpr - 1) / cpr) * G < 2LL * dev_sms) cpr /= 2;
    int h_len = 0;
    int* d_len = nullptr;
    cudaError_t e = cudaMalloc(&d_len, sizeof(int));
    if (e != cudaSuccess) return e;
    for (;;) {
        const int nreg = (c->ncells + cpr - 1) / cpr;
        int32_t* wlo = nullptr;
        e = cudaMalloc(&wlo, sizeof(int32_t) * (size_t)nreg * c->Nd);
        if (e == cudaSuccess) e = cudaMemsetAsync(d_len, 0, sizeof(int), st);
        if (e == cudaSuccess) {
            const int64_t nt = (int64_t)nreg * c->Nd;
            k_mp_windows<<<(unsigned)((nt + 255) / 256), 256, 0, st>>>(c->d_grp, c->ncells, c->d_sens, cpr, nreg, c->k,
                                                                       assa ? 1 : 0, wlo, d_len);
            e = cudaGetLastError();
        }
        if (e == cudaSuccess) e = cudaMemcpyAsync(&h_len, d_len, sizeof(int), cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) {
            cudaFree(wlo);
            cudaFree(d_len);
            why = "gpair_mp.cu: window table";
            return e;
        }
        // ASSA: 4-B rows, blocks start 16-B aligned (up to 3 rows earlier) and span a multiple of 4 rows
        // 32-B rows: blocks start on an 8-row boundary (up to 7 rows earlier; the chunk swizzle)
        const int Lr2 = assa ? (std::max(h_len, 1) + 3 + 3) / 4 * 4 : std::max(h_len, 1) + (c->mp_row == 32 ? 7 : 0);
        if (mp_smem(Lr2, cpr, assa ? 4 : c->mp_row) > 200 * 1024) {
            cudaFree(wlo);
            if (cpr > 1) {
                cpr /= 2;
                continue;
            }
            cudaFree(d_len);
            return cudaSuccess;  // does not fit: the other adjoint kernels
        }
        c->mp_cpr = cpr;
        c->mp_regions = nreg;
        c->mp_Lr2 = Lr2;
        // compile-time slot stride of the 32-B-row kernel (0: runtime), when its ring still fits 3 CTAs
        c->mp_slot = 0;
        if (!assa && c->mp_row == 32) {
            for (int lr : {40, 48, 64, 96})
                if (Lr2 <= lr && mp_smem(lr, cpr, 32) <= 72 * 1024) {
                    c->mp_slot = lr;
                    break;
                }
            if (const char* ev = std::getenv("GPAIR_MP_SLOT_RUNTIME"))
                if (ev[0] == '1') c->mp_slot = 0;  // A/B runs
        }
        c->d_wlo_m = wlo;
        c->workspace_bytes += (int64_t)sizeof(int32_t) * nreg * c->Nd;
        break;
    }
    cudaFree(d_len);
    size_t nM;  // doubles
    if (assa) {  // dconv table [Nd][alpha Nt + 2 pad] fp32, pad a multiple of 4
        c->mp_pad = (c->mp_Lr2 + 4 + 3) / 4 * 4;
        c->mp_NtP = (c->k.alpha * c->Nt + 2 * c->mp_pad + 3) / 4 * 4;  // rows of every sensor start 16-B aligned
        nM = ((size_t)c->Nd * c->mp_NtP + 1) / 2;
    } else {
        c->mp_pad = c->mp_Lr2 + 8;  // zero rows on both sides: every staged block stays inside the table
        c->mp_NtP = c->Nt + W - 1 + 2 * c->mp_pad;
        nM = (size_t)c->Nd * c->mp_NtP * (c->mp_row / 8);
    }
    e = cudaMalloc(&c->d_mp, nM * sizeof(double));
    if (e == cudaSuccess) e = cudaMemsetAsync(c->d_mp, 0, nM * sizeof(double), st);
    if (assa) {
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) {
            why = "gpair_mp.cu: dconv table";
            return e;
        }
        c->workspace_bytes += (int64_t)nM * sizeof(double);
        c->mp_on = 1;
        return cudaSuccess;
    }
    if (e == cudaSuccess) e = cudaMalloc(&c->d_mp_coef, coef.size() * sizeof(double));
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(c->d_mp_coef, coef.data(), coef.size() * sizeof(double), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
        why = "gpair_mp.cu: moment table";
        return e;
    }
    c->workspace_bytes += (int64_t)(nM + coef.size()) * sizeof(double);
    c->mp_on = 1;
    return cudaSuccess;
}

}  // namespace gpair
