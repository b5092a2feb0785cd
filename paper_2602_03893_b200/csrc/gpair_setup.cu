// gpair_setup.cu -- create-time geometry processing.
//
// 1. Spatial sort: kernels are ordered by the Morton code of their grid
//    coordinates (exact integer coordinates when the centres form a regular
//    grid, the paper's voxel lattice P:230; a 1024^3 quantisation otherwise).
//    Consecutive runs of 32 sorted kernels form a "cell" (4x4x2 voxels on a
//    grid).  Each cell gets an fp32 anchor C_c (bounding-box centre) and a
//    conservative radius; each kernel stores delta = c_i - C_c.
// 2. Regions: runs of cells processed by one forward CTA (partial traces) or
//    one adjoint CTA (staged residual windows).  For every (region, sensor)
//    the conservative sample window [lo, hi] of all its pairs is computed in
//    fp64 from the cell anchors and radii (triangle inequality), together with
//    the far-field geometry check r_ij > k sigma (reading R2).
#include <thrust/device_ptr.h>
#include <thrust/execution_policy.h>
#include <thrust/sequence.h>
#include <thrust/sort.h>
#include <thrust/unique.h>

#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "gpair_ctx.h"

namespace gpair {

namespace {

#define SETUP_CHECK(x)                                                   \
    do {                                                                 \
        cudaError_t e_ = (x);                                            \
        if (e_ != cudaSuccess) {                                         \
            if (why.empty()) why = "gpair_setup.cu:" + std::to_string(__LINE__); \
            return e_;                                                   \
        }                                                                \
    } while (0)

__global__ void k_check_finite(const float* __restrict__ c, int64_t n, int* flag) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n && !isfinite(c[i])) atomicOr(flag, 1);
}

__device__ __forceinline__ uint64_t spread3(uint64_t x) {
    x &= 0x1fffffULL;
    x = (x | x << 32) & 0x1f00000000ffffULL;
    x = (x | x << 16) & 0x1f0000ff0000ffULL;
    x = (x | x << 8) & 0x100f00f00f00f00fULL;
    x = (x | x << 4) & 0x10c30c30c30c30c3ULL;
    x = (x | x << 2) & 0x1249249249249249ULL;
    return x;
}

// Morton key of the quantised coordinates; grid mode flags non-integer ones.
__global__ void k_keys(const float* __restrict__ c, int64_t M, double mnx, double mny, double mnz,
                       double stx, double sty, double stz, int grid_mode, uint64_t* keys,
                       int32_t* vals, int* nonint) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= M) return;
    double u[3] = {((double)c[i] - mnx) / stx, ((double)c[M + i] - mny) / sty,
                   ((double)c[2 * M + i] - mnz) / stz};
    uint64_t key = 0;
    for (int a = 0; a < 3; ++a) {
        double q = grid_mode ? rint(u[a]) : floor(u[a]);
        if (grid_mode && fabs(u[a] - q) > 1e-3) atomicOr(nonint, 1);
        q = fmin(fmax(q, 0.0), 2097151.0);
        key |= spread3((uint64_t)q) << a;
    }
    keys[i] = key;
    vals[i] = (int32_t)i;
}

// One warp per 32-kernel cell: fp32 anchors (bounding-box centres) and
// conservative radii of the cell (windows) and of its four 8-kernel groups
// (time-of-flight anchors), and per-kernel offsets from the group anchor.
// Padding lanes (past M) sit on lane 0's kernel with zero amplitude.
__device__ __forceinline__ void bbox_centre(float x, float y, float z, int width, float& Cx, float& Cy,
                                            float& Cz) {
    float mnx = x, mny = y, mnz = z, mxx = x, mxy = y, mxz = z;
    for (int o = width / 2; o > 0; o >>= 1) {
        mnx = fminf(mnx, __shfl_xor_sync(0xffffffffu, mnx, o));
        mny = fminf(mny, __shfl_xor_sync(0xffffffffu, mny, o));
        mnz = fminf(mnz, __shfl_xor_sync(0xffffffffu, mnz, o));
        mxx = fmaxf(mxx, __shfl_xor_sync(0xffffffffu, mxx, o));
        mxy = fmaxf(mxy, __shfl_xor_sync(0xffffffffu, mxy, o));
        mxz = fmaxf(mxz, __shfl_xor_sync(0xffffffffu, mxz, o));
    }
    Cx = (float)(0.5 * ((double)mnx + (double)mxx));
    Cy = (float)(0.5 * ((double)mny + (double)mxy));
    Cz = (float)(0.5 * ((double)mnz + (double)mxz));
}

__device__ __forceinline__ double radius(float x, float y, float z, float Cx, float Cy, float Cz, int width) {
    double dx = (double)x - Cx, dy = (double)y - Cy, dz = (double)z - Cz;
    double rad = sqrt(dx * dx + dy * dy + dz * dz);
    for (int o = width / 2; o > 0; o >>= 1) rad = fmax(rad, __shfl_xor_sync(0xffffffffu, rad, o));
    return rad * (1.0 + 1e-6) + 1e-12;  // conservative margin
}

__global__ void k_cells(const float* __restrict__ c, int64_t M, const int32_t* __restrict__ sorted,
                        int32_t ncells, float4* kd, float4* cell, float4* grp, float* orig, int32_t* perm) {
    int cid = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    int lane = threadIdx.x & 31;
    if (cid >= ncells) return;
    int64_t i = (int64_t)cid * CELL + lane;
    int64_t Mpad = (int64_t)ncells * CELL;
    bool real = i < M;
    int32_t idx = real ? sorted[i] : -1;
    int32_t idx0 = __shfl_sync(0xffffffffu, idx, 0);
    int32_t src = real ? idx : idx0;
    float x = c[src], y = c[M + src], z = c[2 * M + src];
    float Cx, Cy, Cz, Gx, Gy, Gz;
    bbox_centre(x, y, z, CELL, Cx, Cy, Cz);
    bbox_centre(x, y, z, GROUP, Gx, Gy, Gz);
    double crad = radius(x, y, z, Cx, Cy, Cz, CELL);
    double grad = radius(x, y, z, Gx, Gy, Gz, GROUP);
    double dx = (double)x - Gx, dy = (double)y - Gy, dz = (double)z - Gz;
    float fdx = (float)dx, fdy = (float)dy, fdz = (float)dz;
    double d2 = (double)fdx * fdx + (double)fdy * fdy + (double)fdz * fdz;
    kd[i] = make_float4(fdx, fdy, fdz, (float)d2);
    orig[i] = x;
    orig[Mpad + i] = y;
    orig[2 * Mpad + i] = z;
    perm[i] = idx;
    if (lane == 0) cell[cid] = make_float4(Cx, Cy, Cz, (float)crad);
    if ((lane & (GROUP - 1)) == 0) grp[i / GROUP] = make_float4(Gx, Gy, Gz, (float)grad);
}

// fp64 conservative sample window of all pairs of a cell with one sensor.
__device__ __forceinline__ bool cell_window(float4 C, float sx, float sy, float sz, const OpConst& k,
                                            int& lo, int& hi, double& R) {
    double dx = (double)C.x - sx, dy = (double)C.y - sy, dz = (double)C.z - sz;
    R = sqrt(dx * dx + dy * dy + dz * dz);
    double rad = C.w;
    double a = floor(((R - rad - k.win_half) / k.v - k.t0) * k.fs) - 1.0;
    double b = ceil(((R + rad + k.win_half) / k.v - k.t0) * k.fs) + 1.0;
    a = fmax(a, 0.0);
    b = fmin(b, (double)(k.Nt - 1));
    if (a > b) return false;
    lo = (int)a;
    hi = (int)b;
    return true;
}

// Exact far-field geometry test of one cell (reading R2): some pair of the cell has
// r_ij <= k sigma_i, decided with the oracle's fp64 operations (pair_distance:
// differences of the fp32 inputs, sqrt of the sum of squares, no contraction).
__device__ bool cell_pairs_too_close(int cc, const float* __restrict__ orig, const int32_t* __restrict__ perm,
                                     const float4* __restrict__ ksig, int64_t Mpad, float sx, float sy, float sz,
                                     const OpConst& k) {
    for (int t = 0; t < CELL; ++t) {
        const int64_t i = (int64_t)cc * CELL + t;
        if (perm[i] < 0) continue;  // padding
        const double dx = __dsub_rn((double)orig[i], (double)sx);
        const double dy = __dsub_rn((double)orig[Mpad + i], (double)sy);
        const double dz = __dsub_rn((double)orig[2 * Mpad + i], (double)sz);
        const double r = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
        const double ks = ksig ? kernel_ks(ksig[i].z, k) : k.ks;
        if (!(r > ks)) return true;
    }
    return false;
}

// Thread per (region, sensor): union window over the region's cells.
// check != 0 also performs the geometry check and the anchor-expansion bound.
// The geometry check is exact: a cell whose bounding sphere comes within k sigma_max
// of the sensor has its pairs tested one by one (cell_pairs_too_close).
__global__ void k_region_windows(const float4* __restrict__ cell, const float4* __restrict__ grp, int32_t ncells,
                                 const float* __restrict__ sens, int32_t cpr, int32_t nregions,
                                 OpConst k, int32_t* wlo, int* maxlen, int check, int* geom_bad,
                                 unsigned int* max_eps_bits, unsigned int* rmin_bits = nullptr,
                                 unsigned int* rmax_bits = nullptr, const float* __restrict__ orig = nullptr,
                                 const int32_t* __restrict__ perm = nullptr, const float4* __restrict__ ksig = nullptr,
                                 int64_t Mpad = 0) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= (int64_t)nregions * k.Nd) return;
    int j = (int)(t % k.Nd);
    int r = (int)(t / k.Nd);
    float sx = sens[j], sy = sens[k.Nd + j], sz = sens[2 * k.Nd + j];
    int lo = INT_MAX, hi = INT_MIN;
    float eps_max = 0.f;
    float rmin = 3.0e38f, rmax = 0.f;
    int bad = 0;
    int c1 = min((r + 1) * cpr, ncells);
    for (int cc = r * cpr; cc < c1; ++cc) {
        float4 C = cell[cc];
        int a, b;
        double R;
        // union of the four 8-kernel group windows (tighter than the cell sphere)
        for (int gq = 0; gq < GPC; ++gq) {
            double Rg;
            if (cell_window(grp[(int64_t)cc * GPC + gq], sx, sy, sz, k, a, b, Rg)) {
                lo = min(lo, a);
                hi = max(hi, b);
            }
        }
        {
            const double dx = (double)C.x - sx, dy = (double)C.y - sy, dz = (double)C.z - sz;
            R = sqrt(dx * dx + dy * dy + dz * dz);
        }
        if (check) {
            rmin = fminf(rmin, (float)fmax(R - (double)C.w, 0.0));
            rmax = fmaxf(rmax, (float)(R + (double)C.w));
            if (!k.nf && !bad && !(R - (double)C.w > k.ks) &&  // near field: any r > 0 (row f4)
                cell_pairs_too_close(cc, orig, perm, ksig, Mpad, sx, sy, sz, k))
                bad = 1;
            for (int gq = 0; gq < GPC; ++gq) {  // anchor-expansion bound per 8-kernel group
                const float4 G = grp[(int64_t)cc * GPC + gq];
                double gx = (double)G.x - sx, gy = (double)G.y - sy, gz = (double)G.z - sz;
                double Rg2 = gx * gx + gy * gy + gz * gz;
                double e = (2.0 * sqrt(Rg2) * G.w + (double)G.w * G.w) / Rg2;
                eps_max = fmaxf(eps_max, (float)e);
            }
        }
    }
    int len = 0;
    if (lo <= hi) {
        wlo[(int64_t)r * k.Nd + j] = lo;
        len = hi - lo + 1;
    } else {
        wlo[(int64_t)r * k.Nd + j] = -1;
    }
    atomicMax(maxlen, len);
    if (check) {
        if (bad) atomicOr(geom_bad, 1);
        atomicMax(max_eps_bits, __float_as_uint(eps_max));
        if (rmin_bits) atomicMin(rmin_bits, __float_as_uint(rmin));  // non-negative floats order as uints
        if (rmax_bits) atomicMax(rmax_bits, __float_as_uint(rmax));
    }
}

// Forward regions of 512 kernels bound each fp32 partial to ~128 terms per
// sample; when r_max / r_min over the geometry exceeds FWD_WIDE_RATIO (planar
// near-field arrays, cfg5: ~18) the 1/r weights span enough that cancelling
// partials exceed the 1e-4 elementwise bar (measured 1.3e-4 at cfg5), so the
// regions shrink to FWD_CPR_WIDE cells (6.9e-5).
constexpr int FWD_CPR_WIDE = 4;
constexpr float FWD_WIDE_RATIO = 4.f;

// Reducer table (gpair_kernels.cu k_reduce): per sensor j the forward regions
// sorted by window start, as (lo, region) entries.  Regions with an empty
// window (lo = -1) sort first and are skipped.
__global__ void k_reducer_keys(const int32_t* __restrict__ wlo, int32_t nregions, int32_t Nd, int32_t Nt,
                               uint32_t* keys, int32_t* vals) {
    const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= (int64_t)nregions * Nd) return;
    const int32_t r = (int32_t)(idx / Nd), j = (int32_t)(idx - (int64_t)r * Nd);
    keys[idx] = (uint32_t)j * (uint32_t)(Nt + 1) + (uint32_t)(wlo[idx] + 1);
    vals[idx] = r;
}

__global__ void k_reducer_entries(const uint32_t* __restrict__ keys, const int32_t* __restrict__ vals,
                                  int32_t nregions, int32_t Nd, int32_t Nt, int2* ent) {
    const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= (int64_t)nregions * Nd) return;
    const uint32_t j = (uint32_t)(idx / nregions);
    ent[idx] = make_int2((int32_t)(keys[idx] - j * (uint32_t)(Nt + 1)) - 1, vals[idx]);
}

__device__ __forceinline__ int lower_bound_lo(const int2* e, int n, int v) {
    int a = 0, b = n;
    while (a < b) {
        const int m = (a + b) >> 1;
        if (e[m].x < v) a = m + 1; else b = m;
    }
    return a;
}

// thread per sensor: length of the live range [first window start, last + Lf)
__global__ void k_reducer_len(const int2* __restrict__ ent, int32_t nregions, int32_t Nd, int32_t Nt, int32_t Lf,
                              int* jlen_max) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= Nd) return;
    const int2* e = ent + (int64_t)j * nregions;
    const int k0 = lower_bound_lo(e, nregions, 0);
    if (k0 < nregions) atomicMax(jlen_max, min(e[nregions - 1].x + Lf, Nt) - e[k0].x);
}

template <class T>
cudaError_t dmalloc(gpair_ctx* c, T** p, size_t n) {
    size_t bytes = std::max<size_t>(n, 1) * sizeof(T);
    cudaError_t e = cudaMalloc((void**)p, bytes);
    if (e == cudaSuccess) c->workspace_bytes += (int64_t)bytes;
    return e;
}

}  // namespace

cudaError_t build_geometry(gpair_ctx* c, const float* centers, const float* sensors, cudaStream_t st,
                           std::string& why, int& geom_err) {
    geom_err = 0;
    const int64_t M = c->M;
    const int Nd = c->Nd;
    auto pol = thrust::cuda::par.on(st);

    SETUP_CHECK(dmalloc(c, &c->d_flags, 16));
    SETUP_CHECK(dmalloc(c, &c->d_count, 1));
    SETUP_CHECK(cudaMemsetAsync(c->d_flags, 0, 16 * sizeof(int32_t), st));
    SETUP_CHECK(dmalloc(c, &c->d_sens, (size_t)3 * Nd));
    SETUP_CHECK(cudaMemcpyAsync(c->d_sens, sensors, sizeof(float) * 3 * Nd, cudaMemcpyDeviceToDevice, st));
    k_check_finite<<<(unsigned)((3 * M + 255) / 256), 256, 0, st>>>(centers, 3 * M, c->d_flags);
    k_check_finite<<<(unsigned)((3 * Nd + 255) / 256), 256, 0, st>>>(c->d_sens, 3 * Nd, c->d_flags);
    SETUP_CHECK(cudaGetLastError());
    int h_flags[16];
    SETUP_CHECK(cudaMemcpyAsync(h_flags, c->d_flags, sizeof(h_flags), cudaMemcpyDeviceToHost, st));
    SETUP_CHECK(cudaStreamSynchronize(st));
    if (h_flags[0]) {
        why = "non-finite centre or sensor coordinate";
        geom_err = GPAIR_ERR_INVALID_ARGUMENT;
        return cudaSuccess;
    }

    // ---- per-axis unique values -> grid detection
    float* tmp = nullptr;
    SETUP_CHECK(cudaMalloc(&tmp, sizeof(float) * M));
    double mn[3], st3[3];
    int64_t nu[3];
    for (int a = 0; a < 3; ++a) {
        SETUP_CHECK(cudaMemcpyAsync(tmp, centers + a * M, sizeof(float) * M, cudaMemcpyDeviceToDevice, st));
        thrust::device_ptr<float> p(tmp);
        thrust::sort(pol, p, p + M);
        int64_t n = thrust::unique(pol, p, p + M) - p;
        float lo_hi[2];
        SETUP_CHECK(cudaMemcpyAsync(&lo_hi[0], tmp, sizeof(float), cudaMemcpyDeviceToHost, st));
        SETUP_CHECK(cudaMemcpyAsync(&lo_hi[1], tmp + n - 1, sizeof(float), cudaMemcpyDeviceToHost, st));
        SETUP_CHECK(cudaStreamSynchronize(st));
        nu[a] = n;
        mn[a] = lo_hi[0];
        double ext = (double)lo_hi[1] - (double)lo_hi[0];
        st3[a] = ext;  // extent for now
    }
    cudaFree(tmp);
    int grid_mode = (nu[0] * nu[1] * nu[2] == M) ? 1 : 0;
    double step[3];
    double ext_max = std::max(st3[0], std::max(st3[1], st3[2]));
    for (int a = 0; a < 3; ++a) {
        if (grid_mode)
            step[a] = nu[a] > 1 ? st3[a] / (double)(nu[a] - 1) : 1.0;
        else
            step[a] = ext_max > 0 ? ext_max / 1023.0 : 1.0;
    }

    uint64_t* keys = nullptr;
    int32_t* vals = nullptr;
    SETUP_CHECK(cudaMalloc(&keys, sizeof(uint64_t) * M));
    SETUP_CHECK(cudaMalloc(&vals, sizeof(int32_t) * M));
    unsigned nb = (unsigned)((M + 255) / 256);
    k_keys<<<nb, 256, 0, st>>>(centers, M, mn[0], mn[1], mn[2], step[0], step[1], step[2], grid_mode,
                               keys, vals, c->d_flags + 1);
    SETUP_CHECK(cudaGetLastError());
    if (grid_mode) {
        int nonint = 0;
        SETUP_CHECK(cudaMemcpyAsync(&nonint, c->d_flags + 1, sizeof(int), cudaMemcpyDeviceToHost, st));
        SETUP_CHECK(cudaStreamSynchronize(st));
        if (nonint) {
            grid_mode = 0;
            for (int a = 0; a < 3; ++a) step[a] = ext_max > 0 ? ext_max / 1023.0 : 1.0;
            k_keys<<<nb, 256, 0, st>>>(centers, M, mn[0], mn[1], mn[2], step[0], step[1], step[2], 0,
                                       keys, vals, c->d_flags + 1);
            SETUP_CHECK(cudaGetLastError());
        }
    }
    c->grid_detected = grid_mode;
    {
        thrust::device_ptr<uint64_t> kp(keys);
        thrust::device_ptr<int32_t> vp(vals);
        thrust::stable_sort_by_key(pol, kp, kp + M, vp);
    }

    // ---- cells
    c->ncells = (int32_t)((M + CELL - 1) / CELL);
    c->Mpad = (int64_t)c->ncells * CELL;
    SETUP_CHECK(dmalloc(c, &c->d_kd, c->Mpad));
    SETUP_CHECK(dmalloc(c, &c->d_cell, c->ncells));
    SETUP_CHECK(dmalloc(c, &c->d_grp, (size_t)c->ncells * GPC));
    SETUP_CHECK(dmalloc(c, &c->d_orig, 3 * c->Mpad));
    SETUP_CHECK(dmalloc(c, &c->d_perm, c->Mpad));
    k_cells<<<(c->ncells + 7) / 8, 256, 0, st>>>(centers, M, vals, c->ncells, c->d_kd, c->d_cell, c->d_grp,
                                                 c->d_orig, c->d_perm);
    SETUP_CHECK(cudaGetLastError());
    cudaFree(keys);
    cudaFree(vals);
    if (c->gen) {  // per-kernel sigma table and near-field pair lists (row f4, gpair_near.cu)
        SETUP_CHECK(build_general(c, st, why, geom_err));
        if (geom_err) return cudaSuccess;
    }

    // ---- forward regions: sized for >= ~4 CTAs per SM of work and smem fit
    int dev_sms = 148;
    cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, c->device);
    if (c->assa) {
        c->f_warps = std::min(assa_forward_warps(), (Nd + 31) / 32);
        c->f_split = 1;
    } else {  // 8 warps = nsw sensor warps x f_split kernel subsets (split accumulation, k_forward)
        int split = 2;  // measured: 2 -> cfg4 forward rows 5.7e-5 elementwise, 4 costs +1.2 ms
        if (const char* ev = std::getenv("GPAIR_FWD_SPLIT")) split = std::max(1, std::min(8, atoi(ev)));
        while (8 % split) --split;
        const int nsw = std::min(8 / split, (Nd + 31) / 32);
        c->f_warps = 8;
        c->f_split = 8 / nsw;
    }
    c->f_sgroups = (Nd + 32 * (c->f_warps / c->f_split) - 1) / (32 * (c->f_warps / c->f_split));
    int cpr = 16;  // 512 kernels (8x8x8 on a grid): bounds fp32 accumulation chains
    bool cpr_forced = false;
    if (const char* ev = std::getenv("GPAIR_FWD_CPR")) {  // A/B experiments
        cpr = std::max(1, std::min(16, atoi(ev)));
        cpr_forced = true;
    }
    while (cpr > 1 && (int64_t)((c->ncells + cpr - 1) / cpr) * c->f_sgroups < 4LL * dev_sms) cpr /= 2;
    const size_t smem_limit = 220 * 1024;
    for (;;) {
        int nreg = (c->ncells + cpr - 1) / cpr;
        int32_t* wlo = nullptr;
        SETUP_CHECK(cudaMalloc(&wlo, sizeof(int32_t) * (size_t)nreg * Nd));
        SETUP_CHECK(cudaMemsetAsync(c->d_flags + 2, 0, 6 * sizeof(int32_t), st));
        SETUP_CHECK(cudaMemsetAsync(c->d_flags + 8, 0x7f, sizeof(int32_t), st));  // r_min bits (large)
        SETUP_CHECK(cudaMemsetAsync(c->d_flags + 9, 0, sizeof(int32_t), st));     // r_max bits
        int64_t nt = (int64_t)nreg * Nd;
        k_region_windows<<<(unsigned)((nt + 255) / 256), 256, 0, st>>>(
            c->d_cell, c->d_grp, c->ncells, c->d_sens, cpr, nreg, c->k, wlo, c->d_flags + 2, 1, c->d_flags + 3,
            (unsigned int*)(c->d_flags + 4), (unsigned int*)(c->d_flags + 8), (unsigned int*)(c->d_flags + 9),
            c->d_orig, c->d_perm, c->gen ? c->d_ksig : nullptr, c->Mpad);
        SETUP_CHECK(cudaGetLastError());
        SETUP_CHECK(cudaMemcpyAsync(h_flags, c->d_flags, sizeof(h_flags), cudaMemcpyDeviceToHost, st));
        SETUP_CHECK(cudaStreamSynchronize(st));
        if (h_flags[3]) {
            cudaFree(wlo);
            why = "some kernel-sensor distance r_ij <= k*sigma_i: the far-field Eq. 7 model does not apply";
            geom_err = GPAIR_ERR_GEOMETRY;
            return cudaSuccess;
        }
        {
            // accumulation-chain bound: a wide spread of 1/r weights (near-field
            // arrays) makes the fp32 region partials cancel more; use 128-kernel regions there
            float rmn, rmx;
            unsigned b0 = (unsigned)h_flags[8], b1 = (unsigned)h_flags[9];
            memcpy(&rmn, &b0, 4);
            memcpy(&rmx, &b1, 4);
            // the same spread makes the y samples cancel strongly enough that the forward's
            // per-pair scale needs its few-rounding form (measured at cfg5)
            c->tab.pscale = rmx > FWD_WIDE_RATIO * rmn ? 1 : 0;
            if (cpr > FWD_CPR_WIDE && !cpr_forced && rmx > FWD_WIDE_RATIO * rmn) {
                cudaFree(wlo);
                cpr = FWD_CPR_WIDE;
                continue;
            }
        }
        float me;
        unsigned bits = (unsigned)h_flags[4];
        memcpy(&me, &bits, 4);
        c->max_eps = me;
        c->series_small = me <= EPS_SMALL ? 1 : 0;
        {
            const bool cnt_ok = c->k.cnt_int > 0 && pick_wmax(c->k.cnt_int) == c->k.cnt_int;
            c->ser = c->series_small ? (cnt_ok ? 0 : 2) : (cnt_ok ? SER_FAST5 : 5);
        }
        if (c->gen) c->ser = SER_GEN;
        int L = std::max(h_flags[2], 1);
        int Lf = (L + 15) / 16 * 16;  // the flush transposes 32-row blocks plus a 16-row tail
        size_t smem = c->assa ? assa_forward_smem(c, Lf)
                              : (size_t)c->f_warps * Lf * 32 * sizeof(float) + 8 * CELL * (c->gen ? 36 : 20) +
                                    8 * GPC * 16;
        if (smem > smem_limit && cpr > 1) {
            cudaFree(wlo);
            cpr /= 2;
            continue;
        }
        if (smem > smem_limit) {
            cudaFree(wlo);
            why = "per-sensor sample window of a single cell does not fit in shared memory";
            geom_err = GPAIR_ERR_RESOURCE;
            return cudaSuccess;
        }
        c->f_cpr = cpr;
        c->f_regions = nreg;
        c->Lf = Lf;
        c->d_wlo_f = wlo;
        c->workspace_bytes += sizeof(int32_t) * (int64_t)nreg * Nd;
        break;
    }
    {
        // register-window forward (k_forward<16, 0, true>), opt-in with GPAIR_FWD_UNION=1:
        // W = 16 on the degree-2 TAB path of a compact geometry, |2K ln2| * 4 <= 0.6 (its rho polynomial);
        // its register sums keep the fp32 column chains short, so it runs without split accumulation.
        // Measured at cfg4: 46.2 ms against 42.9 ms for the split TAB forward (more accurate: rows
        // 3.8e-5 vs 5.5e-5 elementwise), so it is not the default.
        const char* ev = std::getenv("GPAIR_FWD_UNION");
        c->f_union = (c->k.cnt_int == 16 && c->ser == 0 && c->tab.on && !c->tab.pscale &&
                      std::fabs(c->tab.kappa) * 4.f <= 0.6f && (ev && ev[0] == '1') && !c->assa) ? 1 : 0;
        if (c->f_union) {
            c->f_split = 1;
            c->f_sgroups = (Nd + 32 * c->f_warps - 1) / (32 * c->f_warps);
        }
    }
    // reducer tables (sorted window starts per sensor, chunk ranges)
    {
        const int64_t nt = (int64_t)c->f_regions * Nd;
        uint32_t* keys = nullptr;
        int32_t* vals = nullptr;
        SETUP_CHECK(cudaMalloc(&keys, sizeof(uint32_t) * (size_t)nt));
        SETUP_CHECK(cudaMalloc(&vals, sizeof(int32_t) * (size_t)nt));
        k_reducer_keys<<<(unsigned)((nt + 255) / 256), 256, 0, st>>>(c->d_wlo_f, c->f_regions, Nd, c->Nt, keys, vals);
        SETUP_CHECK(cudaGetLastError());
        thrust::device_ptr<uint32_t> kp(keys);
        thrust::device_ptr<int32_t> vp(vals);
        thrust::stable_sort_by_key(pol, kp, kp + nt, vp);
        SETUP_CHECK(dmalloc(c, &c->d_rent, (size_t)nt));
        k_reducer_entries<<<(unsigned)((nt + 255) / 256), 256, 0, st>>>(keys, vals, c->f_regions, Nd, c->Nt,
                                                                         c->d_rent);
        SETUP_CHECK(cudaGetLastError());
        SETUP_CHECK(cudaStreamSynchronize(st));
        cudaFree(keys);
        cudaFree(vals);
        SETUP_CHECK(cudaMemsetAsync(c->d_flags + 5, 0, sizeof(int32_t), st));
        k_reducer_len<<<(Nd + 127) / 128, 128, 0, st>>>(c->d_rent, c->f_regions, Nd, c->Nt, c->Lf, c->d_flags + 5);
        SETUP_CHECK(cudaGetLastError());
        SETUP_CHECK(cudaMemcpyAsync(h_flags, c->d_flags, sizeof(h_flags), cudaMemcpyDeviceToHost, st));
        SETUP_CHECK(cudaStreamSynchronize(st));
        c->jlen_max = h_flags[5];
    }

    // ---- adjoint regions
    int acpr = 8;
    if (const char* ev = std::getenv("GPAIR_ADJ_CPR")) acpr = std::max(1, std::min(8, atoi(ev)));  // A/B runs
    while (acpr > 1 && (c->ncells + acpr - 1) / acpr < 4 * dev_sms) acpr /= 2;
    for (;;) {
        int nreg = (c->ncells + acpr - 1) / acpr;
        int32_t* wlo = nullptr;
        SETUP_CHECK(cudaMalloc(&wlo, sizeof(int32_t) * (size_t)nreg * Nd));
        SETUP_CHECK(cudaMemsetAsync(c->d_flags + 6, 0, sizeof(int32_t), st));
        int64_t nt = (int64_t)nreg * Nd;
        k_region_windows<<<(unsigned)((nt + 255) / 256), 256, 0, st>>>(
            c->d_cell, c->d_grp, c->ncells, c->d_sens, acpr, nreg, c->k, wlo, c->d_flags + 6, 0, nullptr, nullptr);
        SETUP_CHECK(cudaGetLastError());
        SETUP_CHECK(cudaMemcpyAsync(h_flags, c->d_flags, sizeof(h_flags), cudaMemcpyDeviceToHost, st));
        SETUP_CHECK(cudaStreamSynchronize(st));
        int La = (std::max(h_flags[6], 1) + 3) / 4 * 4;
        size_t smem = (size_t)32 * La * 4 + (size_t)acpr * GPC * 33 * sizeof(Anchor) + 32 * 4;
        if (smem > 96 * 1024 && acpr > 1) {
            cudaFree(wlo);
            acpr /= 2;
            continue;
        }
        if (smem > smem_limit) {
            cudaFree(wlo);
            why = "per-sensor residual window of a cell does not fit in shared memory";
            geom_err = GPAIR_ERR_RESOURCE;
            return cudaSuccess;
        }
        c->a_cpr = acpr;
        c->a_regions = nreg;
        c->La = La;
        c->d_wlo_a = wlo;
        c->workspace_bytes += sizeof(int32_t) * (int64_t)nreg * Nd;
        break;
    }

    // ---- workspaces
    if (c->ser == 0 || c->ser == SER_FAST5) {  // sensor-lane adjoints (k_adjoint_lcf / _t / _sl) group partials
        SETUP_CHECK(dmalloc(c, &c->d_gpart, (size_t)((Nd + 127) / 128) * c->Mpad));  // 128-sensor groups (LCF)
    }
    if ((c->ser == 0 || c->ser == SER_FAST5) && c->tab.on) {
        // lane-centred factorisation tables (k_adjoint_lcf), fp64, tau = t - La/2:
        // Q = 2^{-2K tau}, 1/Q, 1/G, G = 2^{K tau^2}
        const double Kd = -1.4426950408889634 * c->k.h * c->k.h / (2.0 * c->k.sigma * c->k.sigma);
        const int La = c->La, T = La / 2;
        const double tmax = (double)std::max(T, La - T);
        if (std::fabs(Kd) * tmax * tmax <= 100.0) {  // column values delta G stay normal fp32
            std::vector<double> g(4 * (size_t)La);
            for (int t = 0; t < La; ++t) {  // [t][4] = Q, 1/Q, 1/G, G
                const double tau = (double)(t - T);
                g[4 * t] = std::exp2(-2.0 * Kd * tau);
                g[4 * t + 1] = std::exp2(2.0 * Kd * tau);
                g[4 * t + 2] = std::exp2(-Kd * tau * tau);
                g[4 * t + 3] = std::exp2(Kd * tau * tau);
            }
            SETUP_CHECK(dmalloc(c, &c->d_gtab, g.size()));
            SETUP_CHECK(cudaMemcpyAsync(c->d_gtab, g.data(), g.size() * sizeof(double), cudaMemcpyHostToDevice, st));
            SETUP_CHECK(cudaStreamSynchronize(st));
        }
    }
    SETUP_CHECK(dmalloc(c, &c->d_partial, (size_t)c->f_regions * Nd * c->Lf));
    SETUP_CHECK(dmalloc(c, &c->d_amp, c->Mpad));
    SETUP_CHECK(dmalloc(c, &c->d_y, (size_t)Nd * c->Nt));
    SETUP_CHECK(dmalloc(c, &c->d_delta, (size_t)Nd * c->Nt));
    SETUP_CHECK(dmalloc(c, &c->d_loss_part, Nd));
    SETUP_CHECK(mp_setup(c, st, why));  // moment-polynomial adjoint (gpair_mp.cu), when eligible
    SETUP_CHECK(cudaStreamSynchronize(st));
    return cudaSuccess;
}

}  // namespace gpair
