// Microbenchmark: tcgen05.mma issue-to-completion throughput on one SM (cta_group::1,
// kind::f16, bf16 operands, fp32 accumulate in TMEM).  One thread per CTA issues
// `iters` groups of 8 MMAs (K = 8 x 16 = 128) back to back, committing every group to an
// mbarrier and waiting for group g-2 before issuing group g (2 groups in flight),
// then reports cycles per MMA instruction.  Variants: SS (A and B from shared
// memory) with N = 64 / 128 / 256 and TS (A from tensor memory) with N = 128.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../include umma.cu -o umma
#include <cstdio>
#include "../../paper_2503_16525_b200/csrc/common.cuh"

using namespace kvs;

template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) umma_kernel(int iters, long long *cyc) {
    extern __shared__ uint8_t dsmem[];
    __shared__ uint64_t bar[2];
    __shared__ uint32_t tbase;
    const uint32_t base = (smem_u32(dsmem) + 1023u) & ~1023u;
    // A: 128 x 128 bf16 (32 KB, two SW128 halves), B: N x 128 bf16
    const uint32_t sA = base, sB = base + 32768;
    if (threadIdx.x < 32) tmem_alloc(&tbase, 512);
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_barrier_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tbase;
    long long t0 = 0, t1 = 0;
    if (threadIdx.x == 0) {
        const uint32_t idesc = umma_idesc_bf16(128, N, TS);
        t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            if (it >= 2) mbar_wait(&bar[it & 1], (uint32_t)((it >> 1) - 1) & 1u);
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                if constexpr (TS) {
                    const uint64_t db = umma_desc_sw128(sB + k * 2048, 16384, 1024);
                    umma_bf16_ts(tmem + 256, tmem + 8 * k, db, idesc, k > 0 ? 1u : 0u);
                } else {
                    const uint64_t da = umma_desc_sw128(sA + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024);
                    const uint64_t db =
                        umma_desc_sw128(sB + (k >> 2) * (N * 128) + (k & 3) * 32, 16, 1024);
                    umma_bf16(tmem + (it & 1) * 256, da, db, idesc, k > 0 ? 1u : 0u);
                }
            }
            umma_commit(&bar[it & 1]);
        }
        mbar_wait(&bar[(iters - 1) & 1], (uint32_t)(((iters - 1) >> 1)) & 1u);
        t1 = clock64();
        cyc[blockIdx.x] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

template <int N, bool TS>
void run(const char *name, long long *cyc, int grid) {
    const int iters = 2000;
    const size_t smem = 1024 + 32768 + N * 256;
    cudaFuncSetAttribute(umma_kernel<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    umma_kernel<N, TS><<<grid, 128, smem>>>(iters, cyc);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, cyc, sizeof(long long) * grid, cudaMemcpyDeviceToHost);
    const double per = (double)h[0] / (iters * 8.0);
    const double ideal = 128.0 * N * 16 * 2 / 8192.0;     // cycles at 8192 dense bf16 FLOP/clk/SM
    printf("%-12s grid %3d: %.1f cycles per MMA (ideal %.0f, %.0f%%) %s\n", name, grid, per, ideal,
           100.0 * ideal / per, e == cudaSuccess ? "" : cudaGetErrorString(e));
}


// 2-SM variant (cta_group::2): a CTA pair, M = 256 (128 rows per SM), the leader issues.
// A: each CTA's 128 rows at the same shared offset; B: N/2 rows per CTA.
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int N>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) umma2_kernel(int iters, long long *cyc) {
    extern __shared__ uint8_t dsmem[];
    __shared__ uint64_t bar[2];
    __shared__ uint32_t tbase;
    const uint32_t base = (smem_u32(dsmem) + 1023u) & ~1023u;
    const uint32_t sA = base, sB = base + 32768;
    const uint32_t rank = cluster_rank();
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_barrier_init();
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = tbase;
    if (threadIdx.x == 0 && rank == 0) {
        const uint32_t idesc = umma_idesc_bf16(256, N, false);
        const long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            if (it >= 2) mbar_wait(&bar[it & 1], (uint32_t)((it >> 1) - 1) & 1u);
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const uint64_t da = umma_desc_sw128(sA + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024);
                const uint64_t db = umma_desc_sw128(sB + (k >> 2) * (N / 2 * 128) + (k & 3) * 32, 16, 1024);
                asm volatile(
                    "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                    "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem + (it & 1) * 256),
                    "l"(da), "l"(db), "r"(idesc), "r"(k > 0 ? 1u : 0u));
            }
            asm volatile(
                "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                    smem_u32(&bar[it & 1])), "h"((uint16_t)3)
                : "memory");
        }
        mbar_wait(&bar[(iters - 1) & 1], (uint32_t)(((iters - 1) >> 1)) & 1u);
        cyc[blockIdx.x] = clock64() - t0;
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    if (threadIdx.x < 32) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    }
}

template <int N>
void run2(const char *name, long long *cyc, int grid) {
    const int iters = 2000;
    const size_t smem = 1024 + 32768 + N * 256;
    cudaFuncSetAttribute(umma2_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    umma2_kernel<N><<<grid, 128, smem>>>(iters, cyc);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, cyc, sizeof(long long) * grid, cudaMemcpyDeviceToHost);
    const double per = (double)h[0] / (iters * 8.0);
    const double ideal = 128.0 * N * 16 * 2 / 8192.0;     // per SM: 128 rows x N
    printf("%-12s grid %3d: %.1f cycles per MMA (per-SM ideal %.0f, %.0f%%) %s\n", name, grid, per,
           ideal, 100.0 * ideal / per, e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
    long long *cyc;
    cudaMalloc(&cyc, 148 * sizeof(long long));
    for (int grid : {1, 148}) {
        run<64, false>("SS N=64", cyc, grid);
        run<128, false>("SS N=128", cyc, grid);
        run<256, false>("SS N=256", cyc, grid);
        run<128, true>("TS N=128", cyc, grid);
    }
    for (int grid : {2, 148}) {
        run2<128>("2SM M256 N128", cyc, grid);
        run2<256>("2SM M256 N256", cyc, grid);
        run2<64>("2SM M256 N64", cyc, grid);
    }
    return 0;
}
