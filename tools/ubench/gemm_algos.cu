// cuBLASLt algorithm sweep for the step's two projection GEMMs (diagnostic).
// Row-major problems are issued as their column-major transposes:
//   QKV:  qkv[M, 6144] (bf16)          = xb[M, 4096] @ Wqkv[4096, 6144]
//   O:    x[M, 4096]   (fp32, += in place) = o[M, 4096] @ Wo[4096, 4096]  (beta = 1)
// Prints the heuristic's first choice and the fastest of up to 32 candidates.
//   nvcc -O3 -std=c++17 gemm_algos.cu -lcublasLt -o gemm_algos
#include <cublasLt.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <vector>

#define CK(x) do { auto s = (x); if (s != 0) { printf("err %d at %d\n", (int)s, __LINE__); return; } } while (0)

static void sweep(const char *name, int M, int N, int K, bool out_f32, float beta) {
    cublasLtHandle_t lt;
    cublasLtCreate(&lt);
    void *A, *B, *C, *ws;
    const size_t wsz = 64 << 20;
    cudaMalloc(&A, (size_t)M * K * 2);
    cudaMalloc(&B, (size_t)K * N * 2);
    cudaMalloc(&C, (size_t)M * N * (out_f32 ? 4 : 2));
    cudaMalloc(&ws, wsz);
    cudaMemset(A, 0, (size_t)M * K * 2);
    cudaMemset(B, 0, (size_t)K * N * 2);
    cudaMemset(C, 0, (size_t)M * N * (out_f32 ? 4 : 2));
    // column-major view: D^T[N, M] = B^T[N, K] @ A^T[K, M]
    cublasLtMatmulDesc_t op;
    CK(cublasLtMatmulDescCreate(&op, CUBLAS_COMPUTE_32F, CUDA_R_32F));
    cublasLtMatrixLayout_t la, lb, lc;
    CK(cublasLtMatrixLayoutCreate(&la, CUDA_R_16BF, N, K, N));   // B^T
    CK(cublasLtMatrixLayoutCreate(&lb, CUDA_R_16BF, K, M, K));   // A^T
    CK(cublasLtMatrixLayoutCreate(&lc, out_f32 ? CUDA_R_32F : CUDA_R_16BF, N, M, N));
    cublasLtMatmulPreference_t pref;
    CK(cublasLtMatmulPreferenceCreate(&pref));
    CK(cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &wsz,
                                            sizeof(wsz)));
    cublasLtMatmulHeuristicResult_t res[32];
    int n = 0;
    CK(cublasLtMatmulAlgoGetHeuristic(lt, op, la, lb, lc, lc, pref, 32, res, &n));
    const float alpha = 1.f;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const double flop = 2.0 * M * N * K;
    double best = 1e30, first = 0;
    int besti = -1;
    for (int i = 0; i < n; ++i) {
        float ms = 0;
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            for (int it = 0; it < 10; ++it)
                cublasLtMatmul(lt, op, &alpha, B, la, A, lb, &beta, C, lc, C, lc, &res[i].algo, ws,
                               wsz, 0);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
        }
        const double t = ms / 10.0;
        if (i == 0) first = t;
        if (t < best) { best = t; besti = i; }
    }
    printf("%s M=%d N=%d K=%d: %d candidates; heuristic #0 %.3f ms (%.0f TFLOP/s), best #%d %.3f ms "
           "(%.0f TFLOP/s), %.1f%% faster\n", name, M, N, K, n, first, flop / first / 1e9, besti,
           best, flop / best / 1e9, 100.0 * (first - best) / first);
}

int main() {
    sweep("QKV", 19660, 6144, 4096, false, 0.f);
    sweep("O+res", 19660, 4096, 4096, true, 1.f);
    sweep("QKV-all", 32768, 6144, 4096, false, 0.f);
    return 0;
}
