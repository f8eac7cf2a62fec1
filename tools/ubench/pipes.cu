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

__global__ void ex2h2_kernel(float *out, int iters, long long *cyc) {
    // ex2.approx.f16x2: two exponentials per lane per instruction
    unsigned a[8];
    for (int i = 0; i < 8; ++i) a[i] = 0x3c003c00u + threadIdx.x + i;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(a[i]));
    }
    long long t1 = clock64();
    float s = 0.f;
    for (int i = 0; i < 8; ++i) s += (float)(a[i] & 0xff);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void ex2bf2_kernel(float *out, int iters, long long *cyc) {
    // ex2.approx.ftz.bf16x2
    unsigned a[8];
    for (int i = 0; i < 8; ++i) a[i] = 0x3f803f80u + threadIdx.x + i;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(a[i]));
    }
    long long t1 = clock64();
    float s = 0.f;
    for (int i = 0; i < 8; ++i) s += (float)(a[i] & 0xff);
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
        for (int k = 0; k < 4; ++k) {
            long long h[148];
            if (k == 0) ex2_kernel<<<148, warps * 32>>>(out, iters, cyc);
            else if (k == 1) ffma_kernel<<<148, warps * 32>>>(out, iters, cyc);
            else if (k == 2) ex2h2_kernel<<<148, warps * 32>>>(out, iters, cyc);
            else ex2bf2_kernel<<<148, warps * 32>>>(out, iters, cyc);
            cudaDeviceSynchronize();
            cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
            double ops = (double)iters * 8 * warps;           // warp-instructions per SM
            printf("%s warps/SM=%2d: %.2f cycles per warp-instruction per SM  (%.1f lanes/clk/SM)\n",
                   k == 0 ? "EX2.F32 " : k == 1 ? "FFMA    " : k == 2 ? "EX2.F16x2" : "EX2.BF16x2", warps,
                   h[0] / ops, 32.0 * ops / h[0]);
        }
    }
    return 0;
}
