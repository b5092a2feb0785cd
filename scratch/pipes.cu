// microbenchmark: per-SM throughput of DFMA, FFMA, MUFU.EX2 on this GPU
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void k(float* out, int iters) {
    float a = threadIdx.x * 1e-3f, b = 1.0001f, c = 0.999f, d = 0.5f;
    double da = a, db = 1.0000001, dc = 0.9999, dd = 0.3;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            if (OP == 0) { a = fmaf(a, b, c); d = fmaf(d, b, c); }
            if (OP == 1) { da = fma(da, db, dc); dd = fma(dd, db, dc); }
            if (OP == 2) { float r; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a)); a = r * -0.5f; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(d)); d = r*-0.25f; }
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a + d + (float)(da + dd);
}
int main() {
    float* out; cudaMalloc(&out, 148 * 8 * 1024 * 4);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const char* names[] = {"FFMA", "DFMA", "MUFU.EX2(+FMUL)"};
    for (int op = 0; op < 3; ++op) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
            int iters = 4096, blocks = sms * 8, threads = 1024;
            cudaEventRecord(e0);
            if (op == 0) k<0><<<blocks, threads>>>(out, iters);
            if (op == 1) k<1><<<blocks, threads>>>(out, iters);
            if (op == 2) k<2><<<blocks, threads>>>(out, iters);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            double ops = (double)blocks * threads * iters * 16 * 2;
            int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
            if (rep) printf("%s: %.3e ops/s = %.1f ops/clk/SM at %.0f MHz (ms=%.2f)\n", names[op], ops / (ms * 1e-3),
                   ops / (ms * 1e-3) / sms / 1.965e9, 1965.0, ms);
        }
    }
    return 0;
}
