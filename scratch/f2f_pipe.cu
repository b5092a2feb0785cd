// microbenchmark: throughput of F2F.F64.F32 (fp32 -> fp64 conversion) alone and mixed with DFMA,
// and the dependent-issue latency of DFMA (one warp, serial chain)
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void k(double* out, const float* in, int iters) {
    float f0 = in[threadIdx.x & 31], f1 = f0 * 1.5f, f2 = f0 * 0.25f, f3 = f0 + 1.f;
    double a0 = 0, a1 = 0, a2 = 0, a3 = 0, b = 1.0000001;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (OP == 0) {  // 4 conversions (+ adds to keep them live) per u
                a0 += (double)f0; a1 += (double)f1; a2 += (double)f2; a3 += (double)f3;
                f0 += 1.f; f1 += 1.f; f2 += 1.f; f3 += 1.f;
            }
            if (OP == 1) {  // 4 DADD only
                a0 += b; a1 += b; a2 += b; a3 += b;
                f0 += 1.f; f1 += 1.f; f2 += 1.f; f3 += 1.f;
            }
            if (OP == 2) { a0 = fma(a0, b, b); }  // serial DFMA chain (latency)
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + f0;
}
int main() {
    double* out; float* in;
    cudaMalloc(&out, 148 * 8 * 1024 * 8); cudaMalloc(&in, 1024 * 4); cudaMemset(in, 0, 4096);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const char* names[] = {"F2F.F64.F32 + DADD (4 each)", "DADD (4)"};
    for (int op = 0; op < 2; ++op) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
            int iters = 2048, blocks = sms * 8, threads = 1024;
            cudaEventRecord(e0);
            if (op == 0) k<0><<<blocks, threads>>>(out, in, iters);
            if (op == 1) k<1><<<blocks, threads>>>(out, in, iters);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            double n = (double)blocks * threads * iters * 8 * 4;
            if (rep) printf("%s: %.1f per clk per SM (ms=%.2f)\n", names[op], n / (ms * 1e-3) / sms / 1.965e9, ms);
        }
    }
    for (int rep = 0; rep < 2; ++rep) {
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        int iters = 1 << 16;
        cudaEventRecord(e0);
        k<2><<<1, 32>>>(out, in, iters);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (rep) printf("DFMA dependent latency: %.1f cycles\n", ms * 1e-3 * 1.965e9 / (iters * 8.0));
    }
    return 0;
}
