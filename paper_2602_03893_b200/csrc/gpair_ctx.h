// gpair_ctx.h -- host-side context of libgpair (not part of the public ABI).
#pragma once
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "../../include/gpair.h"
#include "gpair_internal.cuh"

struct GpairEventPair {
    int id;
    cudaEvent_t start, stop;
};

struct gpair_ctx_s {
    int device = 0;
    gpair::OpConst k{};
    gpair::TabConst tab{};  // factorised-Gaussian table of the TAB fast path (on = 0: per-sample MUFU path)
    int dbg = 0;            // DBG_* switches (GPAIR_NO_TAB, GPAIR_ADJ_NO_LCF, GPAIR_ADJ_NO_T = 1)
    int64_t M = 0, Mpad = 0;
    int32_t ncells = 0, Nd = 0, Nt = 0;
    int32_t rank = 0, world = 1;
    int coll = 0;           // collective path (world > 1, or GPAIR_COLLECTIVE at world 1)
    void* nccl = nullptr;
    int32_t flags = 0;
    int grid_detected = 0;
    double max_eps = 0.0;
    int series_small = 0;  // 1: every group's |eps| <= EPS_SMALL -> degree-2 series
    int ser = 5;           // kernel path: 0 / SER_FAST5 = packed fast path (degree 2 / 5), 2 / 5 = pair_setup<SER>
    int assa = 0;          // 1: ASSA operator (row f1, gpair_assa.cu)
    float* d_taps = nullptr;   // [2K+1] ASSA taps h[k + K] (fp64-computed, fp32)
    float* d_dconv = nullptr;  // [Nd][alpha Nt] ASSA adjoint correlation buffer

    // geometry in the internal (spatially sorted) order
    float* d_sens = nullptr;   // [3][Nd]
    float4* d_kd = nullptr;    // [Mpad] (dx, dy, dz, |d|^2) relative to the cell anchor
    float4* d_cell = nullptr;  // [ncells] (Cx, Cy, Cz, radius): 32-kernel cell bounds (windows)
    float4* d_grp = nullptr;   // [ncells*4] (Cx, Cy, Cz, radius): 8-kernel group ToF anchors
    float* d_orig = nullptr;   // [3][Mpad] original fp32 centres (exact fp64 window fix-up)
    int32_t* d_perm = nullptr; // [Mpad] sorted -> caller index, -1 = padding

    // forward decomposition
    int32_t f_cpr = 0, f_regions = 0, f_warps = 0, f_sgroups = 0, Lf = 0;
    int32_t f_split = 1;  // kernel subsets per sensor warp in k_forward (split accumulation)
    int32_t f_union = 0;  // 1: register-window forward (k_forward<16, 0, true>)
    int32_t* d_wlo_f = nullptr;   // [f_regions][Nd] window start (-1 = empty)
    int2* d_rent = nullptr;       // [Nd][f_regions] (window start, region) sorted by start (reducer)
    int32_t jlen_max = 0;         // longest per-sensor live range of the partial windows
    int32_t n_loss_part = 0;      // loss partials written by the last reduce / residual launch
    float* d_partial = nullptr;   // [f_regions][Nd][Lf]

    // adjoint decomposition
    int32_t a_cpr = 0, a_regions = 0, La = 0;
    int32_t* d_wlo_a = nullptr;   // [a_regions][Nd]
    gpair::gacc_t* d_gpart = nullptr;     // [ceil(Nd/256)][Mpad] per-sensor-group partial gradients (k_adjoint_t)
    // moment-polynomial adjoint (gpair_mp.cu): regions of mp_cpr cells, start-sample ranges, moments
    int mp_on = 0;
    double mp_fit_err = 0.0;      // max error of the interpolants of the window weights / max |f| (create)
    int32_t mp_row = 48;          // bytes per moment row: 32 (degree 6) or 48 (degree 7)
    int32_t mp_slot = 0;          // compile-time slot stride in rows (40/48/64/96) of k_adjoint_mp, 0: runtime
    int32_t mp_cpr = 0, mp_regions = 0, mp_Lr2 = 0, mp_NtP = 0, mp_pad = 0;
    int32_t* d_wlo_m = nullptr;   // [mp_regions][Nd] lowest n_lo of the region's pairs (INT_MIN: none)
    double* d_mp = nullptr;       // [Nd][mp_NtP][8] fp64 moments M_k[j][n] at row n + W - 1 + mp_pad (chunk-swizzled)
    double* d_mp_coef = nullptr;  // [W][8] interpolation coefficients c_mk
    double* d_gtab = nullptr;     // [La][4] fp64 Q = 2^{-2K tau}, 1/Q, 1/G, G = 2^{K tau^2}, tau = t - La/2 (k_adjoint_lcf), or NULL

    // per-call workspaces
    float* d_amp = nullptr;       // [Mpad] amplitudes in sorted order
    float* d_y = nullptr;         // [Nd][Nt]
    float* d_delta = nullptr;     // [Nd][Nt] residual y - b
    double* d_loss_part = nullptr;// [Nd]
    unsigned long long* d_count = nullptr;
    int32_t* d_flags = nullptr;   // scratch flags

    // general operator (row f4): per-kernel sigma table and near-field pairs
    int gen = 0, nf = 0;
    const float* create_sigmas = nullptr;  // caller's DEVICE sigmas, read during create only
    float4* d_ksig = nullptr;     // [Mpad] (k sigma_i / h, -log2e h^2 / 2 sigma_i^2, sigma_i, 0), sorted order
    int64_t n_near = 0;           // near pairs (r < near_threshold) of this rank
    int32_t n_near_rows = 0, n_near_cols = 0;
    uint64_t* d_near_f = nullptr; // [n_near] (j << 32 | i_sorted), sorted: forward order
    uint64_t* d_near_a = nullptr; // [n_near] (i_sorted << 32 | j), sorted: adjoint order
    int32_t* d_near_rseg = nullptr; // [n_near_rows + 1] segment offsets into d_near_f
    int32_t* d_near_cseg = nullptr; // [n_near_cols + 1] segment offsets into d_near_a
    int32_t* d_near_row = nullptr;  // [Nd] compact near row of sensor j, or -1
    double* d_ynear = nullptr;      // [n_near_rows][Nt] near-field signal rows
    float* d_gnear = nullptr;       // [M] near-field adjoint terms, caller order

    // VCR regulariser workspaces (row f2, gpair_vcr.cu), allocated on first use
    int64_t vcr_M = 0, vcr_Mo = 0; // voxels of the u planes / of the own planes
    int32_t vcr_nb = 0;           // per-block partials of the last launch_vcr_slab
    double* d_vcr_u = nullptr;    // [9][vcr_M] normalised difference fields (fp64)
    double* d_vcr_part = nullptr; // [vcr_nb + 1] per-block fp64 values, then the slab total
    float* d_vcr_g = nullptr;     // [vcr_Mo] dR/dx (caller order)
    float* d_vcr_x = nullptr;     // world > 1: own z planes + halos (NCCL send/recv)
    int64_t vcr_x_n = 0;
    int vcr_prepared = 0;         // gpair_vcr_prepare: slab layout validated on every rank
    int32_t vcr_grid[3] = {0, 0, 0}, vcr_z0 = 0;

    int64_t workspace_bytes = 0;
    std::string err;

    // profiling
    bool prof_on = false;
    int64_t n_launch = 0;  // library kernels launched by per-call entry points (gpair_profile.kernels)
    // sensor-group pipeline of gpair_iterate (gpair_api.cu): launch windows read by the launchers
    int32_t lg0 = 0, lng = 0;   // forward / sensor-lane adjoint: sensor groups [lg0, lg0 + lng) (lng = 0: all)
    int32_t lj0 = 0, lnj = 0;   // reducer / residual: sensors [lj0, lj0 + lnj) (lnj = 0: all)
    bool lskip_gather = false;  // sensor-lane adjoint: leave k_adj_gather to the caller
    cudaStream_t st2 = nullptr; // internal high-priority stream (reducer / collective side of the pipeline)
    cudaEvent_t ev_f[64] = {}, ev_r[64] = {}, ev_fork = nullptr, ev_join = nullptr;
    int pipeline = 0;           // 1: GPAIR_PIPELINE=1 (sensor-group pipeline of gpair_iterate, opt-in)
    std::vector<GpairEventPair> prof_pending;
    std::vector<cudaEvent_t> prof_free;
    double prof_ms[GPAIR_PROF_N] = {0};
    int64_t prof_n[GPAIR_PROF_N] = {0};
};

namespace gpair {

// setup (gpair_setup.cu)
cudaError_t build_geometry(gpair_ctx* c, const float* centers, const float* sensors, cudaStream_t st,
                           std::string& why, int& geom_err);

// kernels (gpair_kernels.cu)
cudaError_t launch_gather(gpair_ctx* c, const float* src, int npc, float eps, cudaStream_t st);
cudaError_t launch_forward(gpair_ctx* c, cudaStream_t st);
cudaError_t launch_reduce(gpair_ctx* c, float* y, const float* b, float* delta, cudaStream_t st);
cudaError_t launch_residual(gpair_ctx* c, const float* y, const float* b, float* delta, cudaStream_t st);
// loss = (1/N) sum of the data partials + lam * sum of n_reg regulariser partials
cudaError_t launch_loss(gpair_ctx* c, float* loss_out, cudaStream_t st, const double* reg_part = nullptr,
                        int32_t n_reg = 0, double lam = 0.0);
struct EpiParams {
    float scale;
    float lr, beta1, beta2, adam_eps, eps_npc, bc1, bc2;
    float* g_out;
    float* z;
    float* m;
    float* v;
    float* x_out;
    const float* g_reg;  // [M] dR/dx in caller order (lam > 0), else NULL
    float lam;
    const float* g_add;  // [M] near-field adjoint terms in caller order (row f4), else NULL
};
enum { EPI_GRAD = 0, EPI_NPC_ADAM = 1, EPI_CLAMP = 2 };

// Adjoint epilogue: g = scale * acc, then either write g,
// or the NPC chain rule (Eq. 19) + bias-corrected Adam,
// or the projected clamp step x <- max(x - lr g, 0); ic = caller index.
template <int MODE>
__device__ __forceinline__ void adjoint_epilogue(float acc, int32_t ic, const EpiParams& ep) {
    if (ep.g_add) acc += ep.g_add[ic];
    const float g = ep.g_reg ? fmaf(ep.lam, ep.g_reg[ic], acc * ep.scale) : acc * ep.scale;
    if (MODE == EPI_GRAD) {
        ep.g_out[ic] = g;
    } else if (MODE == EPI_NPC_ADAM) {
        float z = ep.z[ic];
        const float gz = g * (2.f * (z + ep.eps_npc));
        const float mm = ep.beta1 * ep.m[ic] + (1.f - ep.beta1) * gz;
        const float vv = ep.beta2 * ep.v[ic] + (1.f - ep.beta2) * gz * gz;
        const float mh = mm * ep.bc1, vh = vv * ep.bc2;
        z = z - ep.lr * mh / (sqrtf(vh) + ep.adam_eps);
        ep.z[ic] = z;
        ep.m[ic] = mm;
        ep.v[ic] = vv;
        if (ep.x_out) ep.x_out[ic] = (z + ep.eps_npc) * (z + ep.eps_npc);
    } else {
        const float x = fmaxf(ep.z[ic] - ep.lr * g, 0.f);
        ep.z[ic] = x;
        if (ep.x_out) ep.x_out[ic] = x;
    }
}

cudaError_t launch_adjoint(gpair_ctx* c, const float* resid, int mode, const EpiParams& ep, cudaStream_t st);
cudaError_t launch_count(gpair_ctx* c, cudaStream_t st);
cudaError_t launch_adjoint_gather(gpair_ctx* c, int mode, const EpiParams& ep, cudaStream_t st);
cudaError_t launch_group_gather(gpair_ctx* c, const gacc_t* gpart, int ngroups, int mode, const EpiParams& ep,
                                cudaStream_t st);
int adjoint_groups(const gpair_ctx* c);
int pick_wmax(int w);
// adjoint kernel of a context: 0 = k_adjoint (lane = kernel), 1 = k_adjoint_t (TAB, sensor lanes),
// 2 = k_adjoint_lcf (lane-centred factorisation), 3 = k_adjoint_sl (sensor lanes, per-sample exponential)
// 4 = k_adjoint_mp (lane = kernel, moment polynomial; gpair_mp.cu)
enum { ADJ_LANE_KERNEL = 0, ADJ_TAB_T = 1, ADJ_LCF = 2, ADJ_SL = 3, ADJ_MP = 4 };
int adjoint_kernel(const gpair_ctx* c);
// debug / A-B switches read once at create from the environment
enum { DBG_NO_TAB = 1, DBG_ADJ_NO_LCF = 2, DBG_ADJ_NO_T = 4, DBG_ADJ_NO_MP = 8 };

// moment-polynomial adjoint (gpair_mp.cu)
cudaError_t mp_setup(gpair_ctx* c, cudaStream_t st, std::string& why);
cudaError_t launch_mp_adjoint(gpair_ctx* c, const float* resid, int mode, const EpiParams& ep, cudaStream_t st);
int mp_groups(const gpair_ctx* c);

// ASSA operator (gpair_assa.cu)
size_t assa_forward_smem(const gpair_ctx* c, int Lf);
int assa_forward_warps();
cudaError_t launch_assa_forward(gpair_ctx* c, cudaStream_t st);
cudaError_t launch_assa_adjoint(gpair_ctx* c, const float* resid, int mode, const EpiParams& ep, cudaStream_t st);
cudaError_t launch_assa_count(gpair_ctx* c, cudaStream_t st);
// zero-fill + correlation (Eqs. 15-16) of sensors [j0, j0 + nj) into out[j][pad + q], row stride ld
cudaError_t launch_assa_dconv(gpair_ctx* c, const float* resid, float* out, int64_t ld, int pad, int j0, int nj,
                              cudaStream_t st);

// general operator (gpair_near.cu)
cudaError_t build_general(gpair_ctx* c, cudaStream_t st, std::string& why, int& geom_err);
cudaError_t launch_near_forward(gpair_ctx* c, cudaStream_t st);
cudaError_t launch_near_adjoint(gpair_ctx* c, const float* resid, cudaStream_t st);

// VCR regulariser (gpair_vcr.cu); partial values stay in c->d_vcr_part
cudaError_t vcr_ensure(gpair_ctx* c, int64_t Mu, int64_t Mo);
cudaError_t vcr_slab_ranges(const int32_t* dims, int z0, int nzo, int* zu0, int* zu1, int* zx0, int* zx1);
cudaError_t launch_vcr_slab(gpair_ctx* c, const int32_t* dims, int z0, int nzo, const float* src, int zb, int npc,
                            float eps_npc, float beta, float eps, float* grad, float* value, cudaStream_t st);
cudaError_t launch_vcr_total(gpair_ctx* c, cudaStream_t st);
cudaError_t vcr_slab_ensure(gpair_ctx* c, const int32_t* dims, int z0, int nzo);
cudaError_t launch_vcr(gpair_ctx* c, const int32_t* dims, const float* src, int npc, float eps_npc, float beta,
                       float eps, float* grad, float* value, cudaStream_t st);
inline int32_t vcr_blocks(int64_t M) { return (int32_t)((M + 255) / 256); }

}  // namespace gpair
