// Microbenchmark: issue throughput of MUFU.EX2 vs FFMA per SM on this GPU
// (warps per SM swept).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 pipes.cu -o pipes
#include <cstdio>
#include <cuda_runtime.h>

__global__ void ex2_kernel(float *out, int iters, long long *cyc) {
    float a[8];
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i * 1e-4f;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
    }
    long long t1 = clock64();
    float s = 0.f;
    for (int i = 0; i < 8; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void ffma_kernel(float *out, int iters, long long *cyc) {
    float a[8];
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i * 1e-4f;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32 %0, %0, 0f3F800001, 0f3A000000;" : "+f"(a[i]));
    }
    long long t1 = clock64();
    float s = 0.f;
    for (int i = 0; i < 8; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
    float *out;
    long long *cyc;
    cudaMalloc(&out, 148 * 1024 * 4);
    cudaMalloc(&cyc, 148 * 8);
    const int iters = 4096;
    for (int warps = 1; warps <= 32; warps *= 2) {
        for (int k = 0; k < 2; ++k) {
            long long h[148];
            if (k == 0) ex2_kernel<<<148, warps * 32>>>(out, iters, cyc);
            else ffma_kernel<<<148, warps * 32>>>(out, iters, cyc);
            cudaDeviceSynchronize();
            cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
            double ops = (double)iters * 8 * warps;           // warp-instructions per SM
            printf("%s warps/SM=%2d: %.2f cycles per warp-instruction per SM  (%.1f lanes/clk/SM)\n",
                   k == 0 ? "MUFU.EX2" : "FFMA    ", warps, h[0] / ops, 32.0 * ops / h[0]);
        }
    }
    return 0;
}
