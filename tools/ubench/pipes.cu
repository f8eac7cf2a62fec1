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

// softmax-like mix per element: FFMA (scale, -max), EX2, FADD (row sum),
// half an F2FP (bf16x2 pack), optionally FMNMX (max tracking)
template <int kPack, int kMax>
__global__ void mix_kernel(float *out, int iters, long long *cyc) {
    float s[32];
    for (int i = 0; i < 32; ++i) s[i] = -(threadIdx.x * 1e-3f + i * 1e-2f);
    float l[4] = {0.f, 0.f, 0.f, 0.f}, mx = -1e30f;
    unsigned accs[16] = {0};
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const float mu = 0.5f + (float)it * 1e-7f;           // loop-carried: no hoisting
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
            float x0 = fmaf(s[i], 1.4426950f, -mu), x1 = fmaf(s[i + 1], 1.4426950f, -mu);
            if (kMax) mx = fmaxf(mx, fmaxf(s[i], s[i + 1]));
            float e0, e1;
            asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(e0) : "f"(x0));
            asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(e1) : "f"(x1));
            l[i & 3] += e0;
            l[(i + 1) & 3] += e1;
            if (kPack == 1) {
                unsigned v;
                asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(v) : "f"(e1), "f"(e0));
                accs[i >> 1] ^= v;
            } else if (kPack == 2) {            // round half up + byte permute (ALU)
                const unsigned a = __float_as_uint(e0) + 0x8000u, b = __float_as_uint(e1) + 0x8000u;
                accs[i >> 1] ^= __byte_perm(a, b, 0x7632);
            } else if (kPack == 3) {            // truncation: one byte permute
                accs[i >> 1] ^= __byte_perm(__float_as_uint(e0), __float_as_uint(e1), 0x7632);
            }
        }
    }
    long long t1 = clock64();
    unsigned acc = 0;
    for (int i = 0; i < 16; ++i) acc ^= accs[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = l[0] + l[1] + l[2] + l[3] + (float)acc + mx;
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
    // the mix at 1 and 2 warps per SMSP (cycles per element per SMSP)
    for (int warps = 4; warps <= 8; warps *= 2) {
        for (int v = 0; v < 6; ++v) {
            long long h[148];
            if (v == 0) mix_kernel<0, 0><<<148, warps * 32>>>(out, iters / 8, cyc);
            if (v == 1) mix_kernel<1, 0><<<148, warps * 32>>>(out, iters / 8, cyc);
            if (v == 2) mix_kernel<0, 1><<<148, warps * 32>>>(out, iters / 8, cyc);
            if (v == 3) mix_kernel<1, 1><<<148, warps * 32>>>(out, iters / 8, cyc);
            if (v == 4) mix_kernel<2, 1><<<148, warps * 32>>>(out, iters / 8, cyc);
            if (v == 5) mix_kernel<3, 1><<<148, warps * 32>>>(out, iters / 8, cyc);
            cudaDeviceSynchronize();
            cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
            const double elems = (double)(iters / 8) * 32 * (warps / 4);   // per SMSP
            const int pk = v < 4 ? (v & 1) : v - 2, mxk = v < 4 ? (v >> 1) : 1;
            printf("mix pack=%d max=%d warps/SMSP=%d: %.2f cycles per element-column (EX2 floor 8)\n",
                   pk, mxk, warps / 4, h[0] / elems);
        }
    }
    return 0;
}
