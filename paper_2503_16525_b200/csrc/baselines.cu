// F4 comparison strategies (reference selection.py:133-186): the IDEAL
// leave-one-in deviation scores (the device top-B over given scores,
// kvs_topk_select, lives beside the D2 selectors in dhd.cu).
//
// kvs_ideal_scores: score_i = || attention(q, k + e_i dk, v + e_i dv) -
//   attention(q, k, v) ||_F over heads, rows and dims (selection.py:172-183),
//   without re-running the attention per position: perturbing key/value row
//   i changes row j's softmax only through logit s_ji, so
//     O'_j = (Z_j O_j - e^{s_ji} v_i + e^{s'_ji} (v_i + dv_i)) / (Z_j - e^{s_ji} + e^{s'_ji})
//   with Z_j, O_j of the unperturbed row (all terms shifted by a common max).
//   Pass A: one warp per (head, row) builds m_j, Z_j, O_j.  Pass B: one CTA
//   per (position i, head) accumulates sum_j ||O'_j - O_j||^2 over the rows
//   that see key i.  fp32 throughout; O(H n^2 d) work - a study tool for the
//   reference's small comparison instances, not a serving kernel.
#include "common.cuh"

namespace kvs {

__global__ void __launch_bounds__(256) ideal_base_kernel(const float *__restrict__ q,
                                                         const float *__restrict__ k,
                                                         const float *__restrict__ v, int32_t H,
                                                         int32_t G, int32_t n, int32_t d,
                                                         int32_t causal, float scale,
                                                         float *__restrict__ o,
                                                         float *__restrict__ mz) {
    const int lane = threadIdx.x & 31;
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (w >= (int64_t)H * n) return;
    const int h = (int)(w / n), j = (int)(w % n), g = h / (H / G);
    const float *qj = q + ((int64_t)h * n + j) * d;
    const int kend = causal ? j + 1 : n;
    float m = -INFINITY;
    for (int l = 0; l < kend; ++l) {
        const float *kl = k + ((int64_t)g * n + l) * d;
        float dot = 0.f;
        for (int c = lane; c < d; c += 32) dot += qj[c] * kl[c];
        dot = warp_sum(dot) * scale;
        m = fmaxf(m, dot);
    }
    float z = 0.f;
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};   // d <= 256
    for (int l = 0; l < kend; ++l) {
        const float *kl = k + ((int64_t)g * n + l) * d;
        const float *vl = v + ((int64_t)g * n + l) * d;
        float dot = 0.f;
        for (int c = lane; c < d; c += 32) dot += qj[c] * kl[c];
        const float e = __expf(warp_sum(dot) * scale - m);
        z += e;
#pragma unroll
        for (int t = 0; t < 8; ++t)
            if (lane + 32 * t < d) acc[t] += e * vl[lane + 32 * t];
    }
    float *oj = o + ((int64_t)h * n + j) * d;
#pragma unroll
    for (int t = 0; t < 8; ++t)
        if (lane + 32 * t < d) oj[lane + 32 * t] = acc[t] / z;
    if (lane == 0) {
        mz[2 * ((int64_t)h * n + j)] = m;
        mz[2 * ((int64_t)h * n + j) + 1] = z;
    }
}

__global__ void __launch_bounds__(256) ideal_delta_kernel(
    const float *__restrict__ q, const float *__restrict__ k, const float *__restrict__ v,
    const float *__restrict__ dk, const float *__restrict__ dv, const float *__restrict__ o,
    const float *__restrict__ mz, int32_t H, int32_t G, int32_t n, int32_t d, int32_t causal,
    float scale, float *__restrict__ score2) {
    const int i = blockIdx.x, h = blockIdx.y, g = h / (H / G);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const float *ki = k + ((int64_t)g * n + i) * d, *dki = dk + ((int64_t)g * n + i) * d;
    const float *vi = v + ((int64_t)g * n + i) * d, *dvi = dv + ((int64_t)g * n + i) * d;
    float part = 0.f;
    for (int j = causal ? i + wid : wid; j < n; j += blockDim.x / 32) {
        const float *qj = q + ((int64_t)h * n + j) * d;
        float s = 0.f, sp = 0.f;
        for (int c = lane; c < d; c += 32) {
            s += qj[c] * ki[c];
            sp += qj[c] * (ki[c] + dki[c]);
        }
        s = warp_sum(s) * scale;
        sp = warp_sum(sp) * scale;
        const float m = mz[2 * ((int64_t)h * n + j)], z = mz[2 * ((int64_t)h * n + j) + 1];
        const float M = fmaxf(m, sp);
        const float zs = z * __expf(m - M), es = __expf(s - M), ep = __expf(sp - M);
        const float zp = zs - es + ep;
        const float *oj = o + ((int64_t)h * n + j) * d;
        float sq = 0.f;
        for (int c = lane; c < d; c += 32) {
            const float onew = (zs * oj[c] - es * vi[c] + ep * (vi[c] + dvi[c])) / zp;
            const float del = onew - oj[c];
            sq += del * del;
        }
        part += warp_sum(sq);
    }
    __shared__ float red[8];
    if (lane == 0) red[wid] = part;
    __syncthreads();
    if (threadIdx.x == 0) {
        float t = 0.f;
        for (int w = 0; w < (int)(blockDim.x / 32); ++w) t += red[w];
        atomicAdd(score2 + i, t);
    }
}

__global__ void sqrt_kernel(float *x, int64_t n) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
         t += (int64_t)gridDim.x * blockDim.x)
        x[t] = sqrtf(x[t]);
}

}  // namespace kvs

using namespace kvs;

extern "C" {

size_t kvs_ideal_scores_workspace(int32_t num_heads, int32_t n, int32_t d) {
    return sizeof(float) * ((size_t)num_heads * n * d + 2 * (size_t)num_heads * n + 64);
}

kvs_status kvs_ideal_scores(const float *q, const float *k, const float *v, const float *dk,
                            const float *dv, int32_t num_heads, int32_t kv_heads, int32_t n,
                            int32_t d, int32_t causal, float softmax_scale, float *scores,
                            void *ws, size_t ws_bytes, kvs_stream_t stream) {
    KVS_REQUIRE(num_heads >= 1 && kv_heads >= 1 && num_heads % kv_heads == 0, KVS_ESHAPE,
                "num_heads must be a multiple of kv_heads");
    KVS_REQUIRE(d >= 1 && d <= 256, KVS_ESHAPE, "head dim must be in [1, 256]");
    KVS_REQUIRE(ws_bytes >= kvs_ideal_scores_workspace(num_heads, n, d), KVS_EPARAM,
                "workspace too small");
    if (n <= 0) return KVS_OK;
    cudaStream_t s = (cudaStream_t)stream;
    float *o = (float *)ws;
    float *mz = o + (size_t)num_heads * n * d;
    cudaMemsetAsync(scores, 0, sizeof(float) * n, s);
    const int64_t warps = (int64_t)num_heads * n;
    ideal_base_kernel<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, s>>>(
        q, k, v, num_heads, kv_heads, n, d, causal, softmax_scale, o, mz);
    ideal_delta_kernel<<<dim3(n, num_heads), 256, 0, s>>>(q, k, v, dk, dv, o, mz, num_heads,
                                                          kv_heads, n, d, causal, softmax_scale,
                                                          scores);
    sqrt_kernel<<<(n + 255) / 256, 256, 0, s>>>(scores, n);
    KVS_CHECK_LAUNCH("kvs_ideal_scores");
    return KVS_OK;
}

}  // extern "C"
