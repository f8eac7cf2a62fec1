// Hand-written tcgen05 GEMM for the step's projection shapes, timed beside cuBLAS (diagnostic).
//   C[M, N] (bf16) = A[M, K] @ B[N, K]^T, bf16 in, fp32 accumulator in TMEM.
// Persistent, warp-specialised: warp 0 issues TMA (SW128, 64-element K blocks), warp 1 of
// the leader CTA issues tcgen05.mma into one of two 256-column TMEM accumulators, warps 2-5
// drain the other accumulator (tcgen05.ld -> bf16 -> 32-byte stores) under the next tile's
// main loop.  CG = 1: one SM per 128 x 256 tile.  CG = 2: a CTA pair (cta_group::2) per
// 256 x 256 tile, each SM loading its 128 rows of A and 128 of the 256 rows of B, which
// halves the B traffic per SM.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a gemm_tc.cu -lcublas -o gemm_tc
#include "../../paper_2503_16525_b200/csrc/common.cuh"

#include <cublas_v2.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>

namespace kvs {
bool encode_tmap(CUtensorMap *map, CUtensorMapDataType dtype, int rank, void *gaddr,
                 const uint64_t *dims, const uint64_t *strides_bytes, const uint32_t *box,
                 CUtensorMapSwizzle swz) {
    using Fn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                            const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                            const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                            CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static Fn fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess)
            return false;
        fn = reinterpret_cast<Fn>(p);
    }
    uint32_t estr[5] = {1, 1, 1, 1, 1};
    return fn(map, dtype, rank, gaddr, dims, strides_bytes, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
}  // namespace kvs

using namespace kvs;

namespace gemm {

constexpr int BK = 64;           // K elements per stage (128 bytes: one SW128 row)
constexpr int kThreads = 192;    // warp 0 TMA, warp 1 MMA, warps 2-5 epilogue

template <int CG, int NM>
struct Cfg {
    // NM N=256 MMAs per K step: a CTA pair's tile is 256 x (256 NM); NM = 2 fills all 512
    // TMEM columns (no second accumulator) but halves the operand bytes per FLOP for A
    static constexpr int TN = 256 * NM;
    static constexpr int NBUF = NM == 1 ? 2 : 1;
    static constexpr int N_CTA = TN / CG;        // B rows held by each CTA
    static constexpr int A_BYTES = 128 * 128;
    static constexpr int B_BYTES = N_CTA * 128;
    static constexpr int STAGE = A_BYTES + B_BYTES;
#ifndef STAGES1
#define STAGES1 4
#endif
    static constexpr int STAGES = CG == 2 ? (NM == 2 ? 4 : 6) : STAGES1;
    static constexpr size_t SMEM = 1024 + (size_t)STAGE * STAGES;
};

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::
                     : "memory");
}
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void arrive_expect_cluster(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cluster.shared::cluster.b64 _, [%0], %1;" ::"r"(
                     bar),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void arrive_cluster(uint32_t bar) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar)
                 : "memory");
}
template <int CG>
__device__ __forceinline__ void tma_2d(uint32_t dst, const CUtensorMap *map, uint32_t bar, int c0,
                                       int c1) {
    if constexpr (CG == 2)
        asm volatile(
            "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
            "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1)
            : "memory");
    else
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
            "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1)
            : "memory");
}
template <int CG>
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                    uint32_t acc) {
    if constexpr (CG == 2)
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
            "l"(a), "l"(b), "r"(idesc), "r"(acc));
    else
        umma_bf16(d, a, b, idesc, acc);
}
template <int CG>
__device__ __forceinline__ void commit(uint64_t *bar) {
    if constexpr (CG == 2)
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
            " [%0], %1;" ::"r"(smem_u32(bar)),
            "h"((uint16_t)3)
            : "memory");
    else
        umma_commit(bar);
}

template <int CG, int NM>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                __nv_bfloat16 *__restrict__ C, int M, int N, int K, int mode) {
    // mode 0: GEMM; 1: MMAs on whatever the stages hold, no loads (tensor-pipe rate);
    // 2: loads only (the MMA thread releases each stage as soon as it lands; CG = 1)
    using F = Cfg<CG, NM>;
    extern __shared__ uint8_t dsm[];
    __shared__ uint64_t full[F::STAGES], empty[F::STAGES], acc_full[2], acc_empty[2];
    __shared__ uint32_t tbase;
    const uint32_t base = (smem_u32(dsm) + 1023u) & ~1023u;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = CG == 2 ? cluster_rank() : 0u;
    if (warp == 0) {
        if constexpr (CG == 2) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             smem_u32(&tbase)),
                         "r"(512));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        } else {
            tmem_alloc(&tbase, 512);
        }
    }
    if (threadIdx.x == 32) {
        for (int s = 0; s < F::STAGES; ++s) {
            mbar_init(&full[s], CG);
            mbar_init(&empty[s], mode == 4 ? 2 : 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&acc_full[b], 1);
            mbar_init(&acc_empty[b], 4 * CG);
        }
        fence_barrier_init();
    }
    tc_fence_before();
    __syncthreads();
    if (CG == 2 || mode == 4) cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = tbase;
    const int tiles_n = N / F::TN, n_tiles = (M / (128 * CG)) * tiles_n;
    const int cid = blockIdx.x / CG, ncl = gridDim.x / CG, kblocks = K / BK;

    if (warp == 0) {
        if (lane == 0) {
            tma_prefetch(&ta);
            tma_prefetch(&tb);
            const uint32_t full0 = CG == 2 ? mapa(smem_u32(&full[0]), 0) : smem_u32(&full[0]);
            int it = 0;
            for (int t = cid; t < n_tiles; t += ncl) {
                const int mb = t / tiles_n, nb = t % tiles_n;
                const int arow = mb * 128 * CG + rank * 128;
                const int brow = nb * F::TN + rank * (256 / CG);
                for (int kb = 0; kb < kblocks; ++kb, ++it) {
                    const int s = it % F::STAGES;
                    mbar_wait(&empty[s], ((it / F::STAGES) & 1) ^ 1);
                    const uint32_t fb = full0 + s * 8;
                    const uint32_t sa = base + s * F::STAGE;
                    if (mode == 1) {
                        arrive_cluster(fb);
                        continue;
                    }
                    if (mode == 4) {    // cluster of 2: B split in halves, each multicast to both
                        const uint32_t cr = cluster_rank();
                        arrive_expect_cluster(fb, F::STAGE);
                        tma_2d<1>(sa, &ta, fb, kb * BK, arow);
                        asm volatile(
                            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
                            ".multicast::cluster [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(
                                sa + F::A_BYTES + cr * (F::B_BYTES / 2)),
                            "l"(reinterpret_cast<uint64_t>(&tb)), "r"(fb), "r"(kb * BK),
                            "r"(nb * 256 + (int)cr * 128), "h"((uint16_t)3)
                            : "memory");
                        continue;
                    }
                    if (mode == 3) {    // the same bytes as two contiguous 1-D bulk copies
                        const char *src = reinterpret_cast<const char *>(C) +
                                          ((size_t)(t * kblocks + kb) % 1024) * F::STAGE;
                        arrive_expect_cluster(fb, F::STAGE);
                        asm volatile(
                            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes"
                            " [%0], [%1], %2, [%3];" ::"r"(sa), "l"(src), "r"(F::A_BYTES), "r"(fb)
                            : "memory");
                        asm volatile(
                            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes"
                            " [%0], [%1], %2, [%3];" ::"r"(sa + F::A_BYTES),
                            "l"(src + F::A_BYTES), "r"(F::B_BYTES), "r"(fb)
                            : "memory");
                        continue;
                    }
                    arrive_expect_cluster(fb, F::STAGE);
                    tma_2d<CG>(sa, &ta, fb, kb * BK, arow);
#pragma unroll
                    for (int jj = 0; jj < NM; ++jj)
                        tma_2d<CG>(sa + F::A_BYTES + jj * (256 / CG) * 128, &tb, fb, kb * BK,
                                   brow + jj * 256);
                }
            }
        }
    } else if (warp == 1) {
        if (rank == 0 && lane == 0) {
            const uint32_t idesc = umma_idesc_bf16(128 * CG, 256, false);
            int it = 0, j = 0;
            for (int t = cid; t < n_tiles; t += ncl, ++j) {
                const int buf = j % F::NBUF;
                mbar_wait(&acc_empty[buf], ((j / F::NBUF) & 1) ^ 1);
                tc_fence_after();
                const uint32_t d = tmem + buf * 256;
                for (int kb = 0; kb < kblocks; ++kb, ++it) {
                    const int s = it % F::STAGES;
                    mbar_wait(&full[s], (it / F::STAGES) & 1);
                    tc_fence_after();
                    if (mode >= 2) {
                        mbar_arrive(&empty[s]);
                        if (mode == 4) arrive_cluster(mapa(smem_u32(&empty[s]), cluster_rank() ^ 1));
                        continue;
                    }
                    const uint32_t sa = base + s * F::STAGE, sb = sa + F::A_BYTES;
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k)
#pragma unroll
                        for (int jj = 0; jj < NM; ++jj)
                            mma<CG>(d + jj * 256, umma_desc_sw128(sa + k * 32, 16, 1024),
                                    umma_desc_sw128(sb + jj * (256 / CG) * 128 + k * 32, 16, 1024),
                                    idesc, (kb | k) != 0 ? 1u : 0u);
                    commit<CG>(&empty[s]);
                }
                if (mode >= 2)
                    mbar_arrive(&acc_full[buf]);
                else
                    commit<CG>(&acc_full[buf]);
            }
        }
    } else {
        const int q = warp & 3;    // TMEM lane quarter this warp may access
        const uint32_t empty_bar =
            CG == 2 ? mapa(smem_u32(&acc_empty[0]), 0) : smem_u32(&acc_empty[0]);
        int j = 0;
        for (int t = cid; t < n_tiles; t += ncl, ++j) {
            const int buf = j % F::NBUF;
            const int mb = t / tiles_n, nb = t % tiles_n;
            mbar_wait(&acc_full[buf], (j / F::NBUF) & 1);
            tc_fence_after();
            const int row = mb * 128 * CG + rank * 128 + q * 32 + lane;
            __nv_bfloat16 *dst = C + (size_t)row * N + nb * F::TN;
#pragma unroll 1
            for (int c = 0; c < 8 * NM; ++c) {
                float v[32];
                tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + buf * 256 + c * 32, v);
                tmem_ld_wait();
                uint32_t w[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) w[i] = pack_bf16x2(v[2 * i], v[2 * i + 1]);
                st_global_v8(dst + c * 32, *reinterpret_cast<const uint32_t(*)[8]>(&w[0]));
                st_global_v8(dst + c * 32 + 16, *reinterpret_cast<const uint32_t(*)[8]>(&w[8]));
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) arrive_cluster(empty_bar + buf * 8);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (CG == 2 || mode == 4) cluster_sync_all();
    if (warp == 0) {
        tc_fence_after();
        if constexpr (CG == 2)
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                         "r"(512));
        else
            tmem_dealloc(tmem, 512);
    }
}

template <int CG, int NM = 1>
cudaError_t launch(const CUtensorMap &ta, const CUtensorMap &tb, __nv_bfloat16 *C, int M, int N,
                   int K, int grid, int mode = 0) {
    using F = Cfg<CG, NM>;
    cudaFuncSetAttribute(gemm_kernel<CG, NM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)F::SMEM);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = F::SMEM;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = mode == 4 ? 2 : CG;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, gemm_kernel<CG, NM>, ta, tb, C, M, N, K, mode);
}

}  // namespace gemm

__global__ void fill(__nv_bfloat16 *p, size_t n, uint32_t seed) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x) {
        uint32_t h = (uint32_t)i * 2654435761u ^ seed;
        h ^= h >> 15;
        h *= 2246822519u;
        h ^= h >> 13;
        p[i] = __float2bfloat16(((h & 0xFFFF) / 65536.0f - 0.5f) * 0.25f);
    }
}

static bool make_map(CUtensorMap *m, void *p, int rows, int K, int box_rows) {
    uint64_t dims[2] = {(uint64_t)K, (uint64_t)rows};
    uint64_t strides[1] = {(uint64_t)K * 2};
    uint32_t box[2] = {64, (uint32_t)box_rows};
    return kvs::encode_tmap(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, p, dims, strides, box,
                            CU_TENSOR_MAP_SWIZZLE_128B);
}

template <int CG, int NM = 1>
static void run(const char *name, int M, int N, int K, int reps) {
    __nv_bfloat16 *A, *B, *C, *R;
    cudaMalloc(&A, (size_t)M * K * 2);
    cudaMalloc(&B, (size_t)N * K * 2);
    cudaMalloc(&C, (size_t)M * N * 2);
    cudaMalloc(&R, (size_t)M * N * 2);
    fill<<<1184, 256>>>(A, (size_t)M * K, 1);
    fill<<<1184, 256>>>(B, (size_t)N * K, 2);
    cudaMemset(C, 0, (size_t)M * N * 2);
    CUtensorMap ta, tb;
    if (!make_map(&ta, A, M, K, 128) || !make_map(&tb, B, N, K, 256 / CG)) {
        printf("tensor map failed\n");
        return;
    }
    cublasHandle_t h;
    cublasCreate(&h);
    const float one = 1.f, zero = 0.f;
    auto ref = [&]() {
        cublasGemmEx(h, CUBLAS_OP_T, CUBLAS_OP_N, N, M, K, &one, B, CUDA_R_16BF, K, A, CUDA_R_16BF,
                     K, &zero, R, CUDA_R_16BF, N, CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT);
    };
    const int grid = (148 / CG) * CG;
    cudaError_t e = gemm::launch<CG, NM>(ta, tb, C, M, N, K, grid);
    ref();
    cudaError_t e2 = cudaDeviceSynchronize();
    if (e != cudaSuccess || e2 != cudaSuccess) {
        printf("%s: launch %s / %s\n", name, cudaGetErrorString(e), cudaGetErrorString(e2));
        exit(1);
    }
    std::vector<__nv_bfloat16> hc((size_t)M * N), hr((size_t)M * N);
    cudaMemcpy(hc.data(), C, hc.size() * 2, cudaMemcpyDeviceToHost);
    cudaMemcpy(hr.data(), R, hr.size() * 2, cudaMemcpyDeviceToHost);
    double max_err = 0, max_ref = 0;
    size_t bad = 0;
    for (size_t i = 0; i < hc.size(); ++i) {
        const double a = __bfloat162float(hc[i]), b = __bfloat162float(hr[i]);
        max_err = fmax(max_err, fabs(a - b));
        max_ref = fmax(max_ref, fabs(b));
        if (fabs(a - b) > 1e-2 * fabs(b) + 1e-2) ++bad;
    }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms_mine = 0, ms_ref = 0;
    for (int pass = 0; pass < 2; ++pass) {
        cudaEventRecord(e0);
        for (int r = 0; r < reps; ++r) gemm::launch<CG, NM>(ta, tb, C, M, N, K, grid);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms_mine, e0, e1);
        cudaEventRecord(e0);
        for (int r = 0; r < reps; ++r) ref();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms_ref, e0, e1);
    }
    const double flop = 2.0 * M * N * K;
    float ms_mode[3] = {0, 0, 0};
    for (int mode = 1; mode <= (CG == 1 ? 2 : 1); ++mode) {
        cudaEventRecord(e0);
        for (int r = 0; r < reps; ++r) gemm::launch<CG, NM>(ta, tb, C, M, N, K, grid, mode);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms_mode[mode], e0, e1);
    }
    printf("%-8s   MMA-only %.1f us (%.0f TFLOP/s)   loads-only %.1f us\n", name,
           1e3 * ms_mode[1] / reps, flop * reps / ms_mode[1] / 1e9, 1e3 * ms_mode[2] / reps);
    printf("%-8s M=%d N=%d K=%d  tcgen05 %.1f us (%.0f TFLOP/s)  cuBLAS %.1f us (%.0f TFLOP/s)  "
           "ratio %.3f  max|err| %.3g (max|ref| %.3g, %zu off)\n",
           name, M, N, K, 1e3 * ms_mine / reps, flop * reps / ms_mine / 1e9, 1e3 * ms_ref / reps,
           flop * reps / ms_ref / 1e9, ms_ref / ms_mine, max_err, max_ref, bad);
    cublasDestroy(h);
    cudaFree(A);
    cudaFree(B);
    cudaFree(C);
    cudaFree(R);
}

// Loads-only rate (mode 2, CG = 1) against the number of SMs streaming.
static void probe_loads(int M, int N, int K) {
    __nv_bfloat16 *A, *B, *C;
    cudaMalloc(&A, (size_t)M * K * 2);
    cudaMalloc(&B, (size_t)N * K * 2);
    cudaMalloc(&C, (size_t)M * N * 2);
    CUtensorMap ta, tb;
    make_map(&ta, A, M, K, 128);
    make_map(&tb, B, N, K, 256);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int grid : {2, 8, 38, 74, 148}) {
        // each CTA streams ~the same number of tiles whatever the grid
        const int m = std::min(M, (int)(128 * ((grid * 8 + 23) / 24)));
        float ms = 0;
        for (int pass = 0; pass < 2; ++pass) {
            cudaEventRecord(e0);
            gemm::launch<1>(ta, tb, C, m, N, K, grid, 2);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
        }
        float ms_mc = 0;
        if (grid % 2 == 0) {
            CUtensorMap tb2;
            make_map(&tb2, B, N, K, 128);
            for (int pass = 0; pass < 2; ++pass) {
                cudaEventRecord(e0);
                gemm::launch<1>(ta, tb2, C, m, N, K, grid, 4);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                cudaEventElapsedTime(&ms_mc, e0, e1);
            }
        }
        float ms_bulk = 0;
        for (int pass = 0; pass < 2; ++pass) {
            cudaEventRecord(e0);
            gemm::launch<1>(ta, tb, C, m, N, K, grid, 3);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms_bulk, e0, e1);
        }
        const double bytes = (double)(m / 128) * (N / 256) * (K / 64) * 49152.0;
        printf("loads-only grid %3d: %.2f GB in %.1f us = %.0f GB/s (%.1f B/clk/SM at 1.965 GHz)\n",
               grid, bytes / 1e9, ms * 1e3, bytes / ms / 1e6, bytes / (ms * 1e-3) / grid / 1.965e9);
        printf("   B multicast in CTA pairs grid %3d: %.1f us = %.0f GB/s received (%.1f B/clk/SM)\n",
               grid, ms_mc * 1e3, bytes / ms_mc / 1e6, bytes / (ms_mc * 1e-3) / grid / 1.965e9);
        printf("   1-D bulk copies  grid %3d: %.1f us = %.0f GB/s (%.1f B/clk/SM)\n", grid,
               ms_bulk * 1e3, bytes / ms_bulk / 1e6, bytes / (ms_bulk * 1e-3) / grid / 1.965e9);
    }
}

int main(int argc, char **argv) {
    const int M = argc > 1 ? atoi(argv[1]) : 16384;
    if (argc > 2) {
        probe_loads(M, 6144, 4096);
        return 0;
    }
    const int reps = 20;
    run<1>("1-SM", M, 6144, 4096, reps);
    run<2>("2-SM", M, 6144, 4096, reps);
    run<2, 2>("2-SM x2", M, 6144, 4096, reps);
    run<1>("1-SM", M, 4096, 4096, reps);
    run<2>("2-SM", M, 4096, 4096, reps);
    run<2, 2>("2-SM x2", M, 4096, 4096, reps);
    return 0;
}
