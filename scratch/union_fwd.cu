// Microbenchmark: the forward's inner loop as built ("TAB": 16 in-window
// samples per pair, LDS + FFMA2 + STS into the lane's smem column) against the survey's
// "register window" ("UNION": 8 pairs of a group evaluated at the 22 positions of their
// union window in registers, the in-window mask applied per position, one smem
// read-modify-write per position per group).  Both use the same pair parameters and do
// the arithmetic their designs need per (pair, position); the per-pair time-of-flight set-up
// common to both is left out.  Reports pair-samples (16 per pair) per clock per SM.
#include <cstdio>
#include <cuda_runtime.h>

typedef unsigned long long f2_t;
__device__ __forceinline__ f2_t pk2(float lo, float hi) {
    f2_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void upk2(f2_t v, float& lo, float& hi) { asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v)); }
__device__ __forceinline__ f2_t fma2(f2_t a, f2_t b, f2_t c) {
    f2_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ f2_t mul2(f2_t a, f2_t b) {
    f2_t d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ f2_t add2(f2_t a, f2_t b) {
    f2_t d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}

constexpr int W = 16, C = 8, L = 64, GRP = 8, U = 22;
__constant__ f2_t c2[W / 2], d2[W / 2];

// per pair: (offset k in [0, 6] within the group's union, u_c, P0, r) -- same inputs for both kernels
__global__ void __launch_bounds__(256, 3) k_tab(const float4* __restrict__ prm, int npairs, float* out) {
    extern __shared__ float col[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float* ap0 = col + warp * L * 32 + lane;
    for (int t = 0; t < L; ++t) ap0[t * 32] = 0.f;
    for (int p = 0; p < npairs; p += 2) {
        const int base = (p / GRP) % 4 * 8;  // the group's union start in the column
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const float4 q = prm[(p + h) * 32 + lane];
            float* ap = ap0 + (base + (int)q.x) * 32;
            const f2_t Uc = pk2(q.y, q.y);
            const float r = q.w, r2 = r * r, s = 1.f / r, s2 = s * s;
            f2_t P = pk2(q.z, q.z * r);
#pragma unroll
            for (int i = C; i < W; i += 2) {
                const f2_t Q = fma2(Uc, c2[i / 2], d2[i / 2]);
                f2_t a = pk2(ap[i * 32], ap[(i + 1) * 32]);
                a = fma2(P, Q, a);
                float v0, v1;
                upk2(a, v0, v1);
                ap[i * 32] = v0;
                ap[(i + 1) * 32] = v1;
                P = mul2(P, pk2(r2, r2));
            }
            f2_t Pd = pk2(q.z * s2, q.z * s);
#pragma unroll
            for (int i = C - 2; i >= 0; i -= 2) {
                const f2_t Q = fma2(Uc, c2[i / 2], d2[i / 2]);
                f2_t a = pk2(ap[i * 32], ap[(i + 1) * 32]);
                a = fma2(Pd, Q, a);
                float v0, v1;
                upk2(a, v0, v1);
                ap[i * 32] = v0;
                ap[(i + 1) * 32] = v1;
                Pd = mul2(Pd, pk2(s2, s2));
            }
        }
    }
    __syncwarp();
    float sacc = 0.f;
    for (int t = 0; t < L; ++t) sacc += ap0[t * 32];
    out[blockIdx.x * blockDim.x + threadIdx.x] = sacc;
}

// the register window: positions tau_p = p - U/2 are compile-time; per pair the lane-fixed
// factorisation value_p = alpha rho^tau (tau - a) masked to the pair's 16 positions, summed over
// the group's 8 pairs in registers (position pairs packed in f32x2), then one smem RMW per
// position scaled by the constant G_p
__constant__ f2_t Gp2[U / 2];
__global__ void __launch_bounds__(256, 3) k_union(const float4* __restrict__ prm, int npairs, float* out) {
    extern __shared__ float col[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float* ap0 = col + warp * L * 32 + lane;
    for (int t = 0; t < L; ++t) ap0[t * 32] = 0.f;
    for (int g = 0; g < npairs; g += GRP) {
        f2_t A[U / 2], B[U / 2];
#pragma unroll
        for (int i = 0; i < U / 2; ++i) A[i] = B[i] = 0ull;
#pragma unroll 2
        for (int h = 0; h < GRP; ++h) {
            const float4 q = prm[(g + h) * 32 + lane];
            const int k = (int)q.x;                 // window start within the union
            const float a = q.y + (float)(C + k - U / 2), rho = q.w, rho2 = rho * rho;
            // X_tau = alpha rho^tau from the first position, then x rho^2 per position pair
            f2_t X = pk2(q.z, q.z * rho);
            const f2_t a2 = pk2(a, a);
#pragma unroll
            for (int i = 0; i < U / 2; ++i) {
                const int p0 = 2 * i;
                // in-window masks of positions p0, p0 + 1 (constant except in the 6 + 6 edge positions)
                f2_t Xm = X;
                if (p0 < 6 || p0 + 1 >= W) {  // positions 6..15 are inside every window (k <= 6)
                    const bool m0 = (p0 >= k) && (p0 < k + W), m1 = (p0 + 1 >= k) && (p0 + 1 < k + W);
                    float x0, x1;
                    upk2(X, x0, x1);
                    Xm = pk2(m0 ? x0 : 0.f, m1 ? x1 : 0.f);
                }
                A[i] = add2(A[i], Xm);        // sum alpha rho^tau
                B[i] = fma2(a2, Xm, B[i]);    // sum a alpha rho^tau
                X = mul2(X, pk2(rho2, rho2));
            }
        }
        float* ap = ap0 + ((g / GRP) % 4 * 8) * 32;
#pragma unroll
        for (int i = 0; i < U / 2; ++i) {
            // S_tau = tau A - B, times G_tau, added to the column
            const f2_t tau = pk2((float)(2 * i - U / 2), (float)(2 * i + 1 - U / 2));
            const f2_t S = fma2(tau, A[i], mul2(B[i], pk2(-1.f, -1.f)));
            f2_t c = pk2(ap[2 * i * 32], ap[(2 * i + 1) * 32]);
            c = fma2(S, Gp2[i], c);
            float v0, v1;
            upk2(c, v0, v1);
            ap[2 * i * 32] = v0;
            ap[(2 * i + 1) * 32] = v1;
        }
    }
    __syncwarp();
    float sacc = 0.f;
    for (int t = 0; t < L; ++t) sacc += ap0[t * 32];
    out[blockIdx.x * blockDim.x + threadIdx.x] = sacc;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int npairs = 4096, threads = 256, blocks = sms * 3 * 8;
    float4* prm;
    float* out;
    cudaMalloc(&prm, sizeof(float4) * npairs * 32);
    cudaMalloc(&out, sizeof(float) * blocks * threads);
    {
        float4* h = new float4[npairs * 32];
        unsigned s = 1;
        for (int i = 0; i < npairs * 32; ++i) {
            s = s * 1664525u + 1013904223u;
            h[i] = make_float4((float)(s % 7), -((s >> 8) % 1000) / 1000.f, 1.f, 1.f + ((s >> 16) % 100) * 1e-3f);
        }
        cudaMemcpy(prm, h, sizeof(float4) * npairs * 32, cudaMemcpyHostToDevice);
        delete[] h;
        f2_t z[U / 2];
        for (int i = 0; i < U / 2; ++i) z[i] = 0x3f8000003f800000ull;
        cudaMemcpyToSymbol(c2, z, sizeof(f2_t) * W / 2);
        cudaMemcpyToSymbol(d2, z, sizeof(f2_t) * W / 2);
        cudaMemcpyToSymbol(Gp2, z, sizeof(f2_t) * U / 2);
    }
    const size_t smem = 8 * L * 32 * 4;
    cudaFuncSetAttribute(k_tab, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_union, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const char* names[2] = {"TAB (as built: LDS+FFMA2+STS per sample)", "UNION (register window, 22 positions)"};
    for (int kk = 0; kk < 2; ++kk) {
        for (int rep = 0; rep < 3; ++rep) {
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0);
            if (kk == 0) k_tab<<<blocks, threads, smem>>>(prm, npairs, out);
            else k_union<<<blocks, threads, smem>>>(prm, npairs, out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double ps = (double)blocks * threads * npairs * W;  // useful pair-samples
            if (rep == 2)
                printf("%-44s %.2f ms  %.2f pair-samples/clk/SM (at 1965 MHz)\n", names[kk], ms,
                       ps / (ms * 1e-3) / sms / 1.965e9);
        }
    }
    cudaError_t e = cudaGetLastError();
    printf("status %s\n", cudaGetErrorString(e));
    return 0;
}
