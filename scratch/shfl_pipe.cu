// Microbenchmark: does SHFL consume shared-memory (l1tex data pipe) wavefronts?
#include <cstdio>
__global__ void k_shfl(float* out, int n) {
    float a = threadIdx.x, s = 0.f;
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) s += __shfl_sync(0xffffffffu, a, (i + u) & 31);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_lds(float* out, int n) {
    __shared__ float sm[256];
    sm[threadIdx.x] = threadIdx.x;
    __syncthreads();
    float s = 0.f;
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) s += sm[(threadIdx.x & ~31) + ((i + u) & 31)];
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    float* d; cudaMalloc(&d, 148 * 8 * 256 * 4);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int rep = 0; rep < 2; ++rep) {
        float ms;
        cudaEventRecord(a); k_shfl<<<148 * 8, 256>>>(d, 4096); cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("shfl: %.3f ms -> %.2f warp-shfl/clk/SM at 1.965GHz\n", ms, 148.0 * 8 * 8 * 4096 * 8 / (ms * 1e-3) / 148 / 1.965e9);
        cudaEventRecord(a); k_lds<<<148 * 8, 256>>>(d, 4096); cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("lds : %.3f ms -> %.2f warp-lds/clk/SM\n", ms, 148.0 * 8 * 8 * 4096 * 8 / (ms * 1e-3) / 148 / 1.965e9);
    }
    return 0;
}
