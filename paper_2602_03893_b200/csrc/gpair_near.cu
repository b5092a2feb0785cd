// gpair_near.cu -- the general operator of SURVEY 8f row f4:
//   * per-kernel sigma_i: table d_ksig (sorted order) read by the SER_GEN
//     paths of k_forward / k_adjoint (gpair_kernels.cu, pair_gen);
//   * near field (GPAIR_NEAR_FIELD): Eq. 6 with both
//     terms, each truncated to |.| < k sigma_i (reading N1).  Pairs with
//     r < near_threshold (k sigma_i + max(0, -v t0), plus a margin) are
//     "near": the main kernels skip them and the kernels below evaluate
//     both terms in fp64 with the oracle's operation order, so window
//     membership is decided bit-identically.  Every other pair's incoming
//     window is empty (d+ = r + v t_n >= r + v t0 >= k sigma_i).
// Near pairs are rare (a sensor inside or touching the kernel volume), so
// these kernels are plain one-thread-per-segment loops; determinism comes
// from sorting the pair lists.
#include <thrust/execution_policy.h>
#include <thrust/scan.h>
#include <thrust/sort.h>

#include "gpair_ctx.h"

namespace gpair {

namespace {

constexpr uint64_t LO32 = 0xffffffffull;

__global__ void k_ksig(const float* __restrict__ sig_in, const int32_t* __restrict__ perm, int64_t Mpad, OpConst k,
                       float sig_pad, float4* __restrict__ ksig) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= Mpad) return;
    const int32_t ic = perm[i];
    const float sf = sig_in ? (ic >= 0 ? sig_in[ic] : sig_pad) : (float)k.sigma;
    const double s = k.per_sigma ? (double)sf : k.sigma;
    const double ks = k.per_sigma ? k.kwin * s : k.ks;
    const double log2e = 1.4426950408889634;
    ksig[i] = make_float4((float)(ks / k.h), (float)(-log2e * k.h * k.h / (2.0 * s * s)), sf, 0.f);
}

// Thread per (cell, sensor): emit the near pairs (j << 32 | i_sorted).
__global__ void k_near_scan(const float4* __restrict__ cell, const float* __restrict__ orig,
                            const float4* __restrict__ ksig, const int32_t* __restrict__ perm,
                            const float* __restrict__ sens, int32_t ncells, int64_t Mpad, OpConst k,
                            unsigned long long* counter, uint64_t* out, int64_t cap, int* zero_r) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= (int64_t)ncells * k.Nd) return;
    const int j = (int)(t % k.Nd);
    const int cc = (int)(t / k.Nd);
    const float sx = sens[j], sy = sens[k.Nd + j], sz = sens[2 * k.Nd + j];
    const float4 C = cell[cc];
    const double dx = (double)C.x - sx, dy = (double)C.y - sy, dz = (double)C.z - sz;
    if (sqrt(dx * dx + dy * dy + dz * dz) - (double)C.w > k.nf_thr_max) return;
    for (int l = 0; l < CELL; ++l) {
        const int64_t i = (int64_t)cc * CELL + l;
        if (perm[i] < 0) continue;
        const double r = exact_r(orig[i], orig[Mpad + i], orig[2 * Mpad + i], sx, sy, sz);
        if (!(r > 0.0)) atomicOr(zero_r, 1);
        if (r < near_threshold(kernel_ks(ksig[i].z, k), k)) {
            const unsigned long long q = atomicAdd(counter, 1ull);
            if ((int64_t)q < cap) out[q] = ((uint64_t)j << 32) | (uint64_t)i;
        }
    }
}

__global__ void k_swap_key(const uint64_t* __restrict__ in, int64_t n, uint64_t* __restrict__ out) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p < n) out[p] = (in[p] << 32) | (in[p] >> 32);
}

__global__ void k_heads(const uint64_t* __restrict__ key, int64_t n, int32_t* __restrict__ flag) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p < n) flag[p] = (p == 0 || (key[p] >> 32) != (key[p - 1] >> 32)) ? 1 : 0;
}

// seg[pos[p]] = p at every head; row_of[hi(key)] = pos[p] (forward list only)
__global__ void k_segments(const uint64_t* __restrict__ key, int64_t n, const int32_t* __restrict__ flag,
                           const int32_t* __restrict__ pos, int32_t* __restrict__ seg, int32_t nseg,
                           int32_t* __restrict__ row_of) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p < n && flag[p]) {
        seg[pos[p]] = (int32_t)p;
        if (row_of) row_of[key[p] >> 32] = pos[p];
    }
    if (p == 0) seg[nseg] = (int32_t)n;
}

// Candidate samples of both terms (the oracle's nf_range, generous by 2).
__device__ __forceinline__ void nf_range(double r, double ks, const OpConst& k, int& n0, int& n1) {
    double lo = floor(((r - ks) / k.v - k.t0) * k.fs) - 2.0;
    double hi = ceil(((r + ks) / k.v - k.t0) * k.fs) + 2.0;
    const double lo2 = floor(((-ks - r) / k.v - k.t0) * k.fs) - 2.0;
    const double hi2 = ceil(((ks - r) / k.v - k.t0) * k.fs) + 2.0;
    lo = fmax(lo, 0.0);
    hi = fmin(hi, (double)(k.Nt - 1));
    if (fmax(lo2, 0.0) <= fmin(hi2, (double)(k.Nt - 1))) {
        lo = fmin(lo, fmax(lo2, 0.0));
        hi = fmax(hi, fmin(hi2, (double)(k.Nt - 1)));
    }
    n0 = (int)lo;
    n1 = (int)hi;
}

// a_ijn of reading N1 with the oracle's operation order (no contraction).
__device__ __forceinline__ double nf_entry(double r, double s, double ks, int n, const OpConst& k) {
    const double t = __dadd_rn(k.t0, __ddiv_rn((double)n, k.fs));
    const double vt = __dmul_rn(k.v, t);
    const double dm = __dsub_rn(r, vt), dp = __dadd_rn(r, vt);
    const double s2 = __dmul_rn(__dmul_rn(2.0, s), s);
    double tm = 0.0, tp = 0.0;
    if (fabs(dm) < ks) tm = __dmul_rn(dm, exp(__ddiv_rn(-__dmul_rn(dm, dm), s2)));
    if (fabs(dp) < ks) tp = __dmul_rn(dp, exp(__ddiv_rn(-__dmul_rn(dp, dp), s2)));
    return __ddiv_rn(__dadd_rn(tm, tp), __dmul_rn(2.0, r));
}

// Thread per near sensor row: ynear[row][n] = sum over its near pairs.
__global__ void k_near_forward(const uint64_t* __restrict__ key, const int32_t* __restrict__ seg, int32_t nseg,
                               const float* __restrict__ orig, const float4* __restrict__ ksig,
                               const float* __restrict__ amp, const float* __restrict__ sens, int64_t Mpad,
                               OpConst k, double* __restrict__ ynear) {
    const int rr = blockIdx.x * blockDim.x + threadIdx.x;
    if (rr >= nseg) return;
    double* row = ynear + (int64_t)rr * k.Nt;
    for (int n = 0; n < k.Nt; ++n) row[n] = 0.0;
    const int p0 = seg[rr], p1 = seg[rr + 1];
    const int j = (int)(key[p0] >> 32);
    const float sx = sens[j], sy = sens[k.Nd + j], sz = sens[2 * k.Nd + j];
    for (int p = p0; p < p1; ++p) {
        const int64_t i = (int64_t)(key[p] & LO32);
        const double A = (double)amp[i];
        if (A == 0.0) continue;
        const float sf = ksig[i].z;
        const double s = kernel_sigma(sf, k), ks = kernel_ks(sf, k);
        const double r = exact_r(orig[i], orig[Mpad + i], orig[2 * Mpad + i], sx, sy, sz);
        int n0, n1;
        nf_range(r, ks, k, n0, n1);
        for (int n = n0; n <= n1; ++n) row[n] += A * nf_entry(r, s, ks, n, k);
    }
}

// Thread per kernel with near pairs: gnear[caller i] = sum_j sum_n a_ijn delta_j[n].
__global__ void k_near_adjoint(const uint64_t* __restrict__ key, const int32_t* __restrict__ seg, int32_t nseg,
                               const float* __restrict__ orig, const float4* __restrict__ ksig,
                               const int32_t* __restrict__ perm, const float* __restrict__ sens,
                               const float* __restrict__ resid, int64_t Mpad, OpConst k, float* __restrict__ gnear) {
    const int cc = blockIdx.x * blockDim.x + threadIdx.x;
    if (cc >= nseg) return;
    const int p0 = seg[cc], p1 = seg[cc + 1];
    const int64_t i = (int64_t)(key[p0] >> 32);
    const float sf = ksig[i].z;
    const double s = kernel_sigma(sf, k), ks = kernel_ks(sf, k);
    double acc = 0.0;
    for (int p = p0; p < p1; ++p) {
        const int j = (int)(key[p] & LO32);
        const double r = exact_r(orig[i], orig[Mpad + i], orig[2 * Mpad + i], sens[j], sens[k.Nd + j],
                                 sens[2 * k.Nd + j]);
        const float* dj = resid + (int64_t)j * k.Nt;
        int n0, n1;
        nf_range(r, ks, k, n0, n1);
        for (int n = n0; n <= n1; ++n) acc += nf_entry(r, s, ks, n, k) * (double)dj[n];
    }
    gnear[perm[i]] = (float)acc;
}

cudaError_t make_segments(gpair_ctx* c, const uint64_t* key, int64_t n, int32_t** seg, int32_t* nseg,
                          int32_t* row_of, cudaStream_t st) {
    int32_t *flag = nullptr, *pos = nullptr;
    cudaError_t e = cudaMalloc(&flag, sizeof(int32_t) * n);
    if (e == cudaSuccess) e = cudaMalloc(&pos, sizeof(int32_t) * n);
    const unsigned nb = (unsigned)((n + 255) / 256);
    if (e == cudaSuccess) {
        k_heads<<<nb, 256, 0, st>>>(key, n, flag);
        thrust::exclusive_scan(thrust::cuda::par.on(st), flag, flag + n, pos);
        int32_t last[2];
        e = cudaMemcpyAsync(&last[0], pos + n - 1, 4, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaMemcpyAsync(&last[1], flag + n - 1, 4, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e == cudaSuccess) {
            *nseg = last[0] + last[1];
            e = cudaMalloc(seg, sizeof(int32_t) * (*nseg + 1));
            c->workspace_bytes += sizeof(int32_t) * (*nseg + 1);
        }
        if (e == cudaSuccess) {
            k_segments<<<nb, 256, 0, st>>>(key, n, flag, pos, *seg, *nseg, row_of);
            e = cudaGetLastError();
        }
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    }
    cudaFree(flag);
    cudaFree(pos);
    return e;
}

}  // namespace

// Per-kernel sigma table and, with the near-field flag, the near-pair lists.
// Called by build_geometry after the cells exist.  geom_err = GEOMETRY when
// some pair has r = 0 (reading N3).
#define NEAR_TAG(e)                                                           \
    do {                                                                      \
        if ((e) != cudaSuccess && why.empty()) why = "gpair_near.cu:" + std::to_string(__LINE__); \
    } while (0)

cudaError_t build_general(gpair_ctx* c, cudaStream_t st, std::string& why, int& geom_err) {
    const int64_t Mpad = c->Mpad;
    cudaError_t e = cudaMalloc(&c->d_ksig, sizeof(float4) * Mpad);
    if (e != cudaSuccess) { NEAR_TAG(e); return e; }
    c->workspace_bytes += sizeof(float4) * Mpad;
    float sig_pad = (float)c->k.sigma;
    if (c->create_sigmas) {  // any valid sigma for the padding lanes (amplitude 0 / never written)
        e = cudaMemcpyAsync(&sig_pad, c->create_sigmas, sizeof(float), cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) { NEAR_TAG(e); return e; }
    }
    k_ksig<<<(unsigned)((Mpad + 255) / 256), 256, 0, st>>>(c->create_sigmas, c->d_perm, Mpad, c->k, sig_pad, c->d_ksig);
    e = cudaGetLastError();
    if (e != cudaSuccess || !c->nf) { NEAR_TAG(e); return e; }

    unsigned long long* counter = (unsigned long long*)c->d_count;
    int* zero_r = c->d_flags + 7;
    const int64_t nt = (int64_t)c->ncells * c->Nd;
    const unsigned nb = (unsigned)((nt + 255) / 256);
    e = cudaMemsetAsync(counter, 0, sizeof(unsigned long long), st);
    if (e == cudaSuccess) e = cudaMemsetAsync(zero_r, 0, sizeof(int), st);
    if (e != cudaSuccess) { NEAR_TAG(e); return e; }
    k_near_scan<<<nb, 256, 0, st>>>(c->d_cell, c->d_orig, c->d_ksig, c->d_perm, c->d_sens, c->ncells, Mpad, c->k,
                                    counter, nullptr, 0, zero_r);
    unsigned long long cnt = 0;
    int hz = 0;
    e = cudaMemcpyAsync(&cnt, counter, sizeof(cnt), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&hz, zero_r, sizeof(int), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) { NEAR_TAG(e); return e; }
    if (hz) {
        why = "some kernel-sensor distance r_ij is 0 (Eq. 6 is singular there)";
        geom_err = GPAIR_ERR_GEOMETRY;
        return cudaSuccess;
    }
    if (cnt >= (1ull << 31)) {
        why = "more than 2^31 near-field pairs";
        geom_err = GPAIR_ERR_RESOURCE;
        return cudaSuccess;
    }
    c->n_near = (int64_t)cnt;
    e = cudaMalloc(&c->d_gnear, sizeof(float) * c->M);
    if (e == cudaSuccess) e = cudaMemsetAsync(c->d_gnear, 0, sizeof(float) * c->M, st);
    if (e == cudaSuccess) e = cudaMalloc(&c->d_near_row, sizeof(int32_t) * c->Nd);
    if (e == cudaSuccess) e = cudaMemsetAsync(c->d_near_row, 0xff, sizeof(int32_t) * c->Nd, st);  // -1
    if (e != cudaSuccess) { NEAR_TAG(e); return e; }
    c->workspace_bytes += sizeof(float) * c->M + sizeof(int32_t) * c->Nd;
    if (cnt == 0) return cudaSuccess;
    e = cudaMalloc(&c->d_near_f, sizeof(uint64_t) * cnt);
    if (e == cudaSuccess) e = cudaMalloc(&c->d_near_a, sizeof(uint64_t) * cnt);
    if (e == cudaSuccess) e = cudaMemsetAsync(counter, 0, sizeof(unsigned long long), st);
    if (e != cudaSuccess) { NEAR_TAG(e); return e; }
    c->workspace_bytes += 2 * sizeof(uint64_t) * cnt;
    k_near_scan<<<nb, 256, 0, st>>>(c->d_cell, c->d_orig, c->d_ksig, c->d_perm, c->d_sens, c->ncells, Mpad, c->k,
                                    counter, c->d_near_f, (int64_t)cnt, zero_r);
    e = cudaGetLastError();
    if (e != cudaSuccess) { NEAR_TAG(e); return e; }
    const int64_t n = (int64_t)cnt;
    thrust::sort(thrust::cuda::par.on(st), c->d_near_f, c->d_near_f + n);
    k_swap_key<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(c->d_near_f, n, c->d_near_a);
    thrust::sort(thrust::cuda::par.on(st), c->d_near_a, c->d_near_a + n);
    e = make_segments(c, c->d_near_f, n, &c->d_near_rseg, &c->n_near_rows, c->d_near_row, st);
    if (e == cudaSuccess) e = make_segments(c, c->d_near_a, n, &c->d_near_cseg, &c->n_near_cols, nullptr, st);
    if (e == cudaSuccess) e = cudaMalloc(&c->d_ynear, sizeof(double) * (size_t)c->n_near_rows * c->Nt);
    if (e == cudaSuccess) c->workspace_bytes += sizeof(double) * (int64_t)c->n_near_rows * c->Nt;
    NEAR_TAG(e);
    return e;
}

cudaError_t launch_near_forward(gpair_ctx* c, cudaStream_t st) {
    if (!c->n_near) return cudaSuccess;
    ++c->n_launch;
    k_near_forward<<<(c->n_near_rows + 63) / 64, 64, 0, st>>>(c->d_near_f, c->d_near_rseg, c->n_near_rows, c->d_orig,
                                                             c->d_ksig, c->d_amp, c->d_sens, c->Mpad, c->k,
                                                             c->d_ynear);
    return cudaGetLastError();
}

cudaError_t launch_near_adjoint(gpair_ctx* c, const float* resid, cudaStream_t st) {
    if (!c->n_near) return cudaSuccess;
    ++c->n_launch;
    k_near_adjoint<<<(c->n_near_cols + 63) / 64, 64, 0, st>>>(c->d_near_a, c->d_near_cseg, c->n_near_cols, c->d_orig,
                                                             c->d_ksig, c->d_perm, c->d_sens, resid, c->Mpad, c->k,
                                                             c->d_gnear);
    return cudaGetLastError();
}

}  // namespace gpair
