// P1 - decode-size projections (model.py:193-195 QKV, model.py:202 output + residual add) for
// row counts up to 64: a decode token step multiplies 8-64 rows by every layer's weights, so
// the step is bound by streaming the weights once from HBM, and the library GEMM reaches
// 0.4-0.57 of that.  Measured (profiles/r2_p1_skinny.txt): faster than the library GEMM only
// at 8 rows for the output projection, slower at the decode step's 32 rows, so the engine
// uses it only with KVS_SKINNY_PROJ=1.
//
// out[m, n] = x[m, k] @ W[k, n] with W packed as 16 x 64 tiles of its transpose,
// w_p[n/16][k/64][16][64] (element (i, j) of W at [j/16][i/64][j%16][i%64]): each
// warp-iteration reads one contiguous 2 KB tile.  A cluster of 8 CTAs owns 128 output
// columns; CTA rank c takes the k-slice [c*k/8, (c+1)*k/8) and each of its 8 warps streams
// the tiles of its 16 columns over the slice (the next tile's loads in flight under this
// one's MMAs).  The tile rows (output columns) are the M side of mma.sync m16n8k16 and the
// x rows the N side, so m <= 64 costs at most 8 MMAs per k16 step.  Inside each 32-k chunk
// lane t holds k [8t, 8t+8) of its two rows, i.e. the chunk's k order is permuted; x is read with the same
// permutation, which leaves the dot products unchanged.  The 8 k-slice partials meet in
// distributed shared memory: rank c sums columns [16c, 16c+16) over the cluster in rank
// order (deterministic) and applies the epilogue (bf16 store, or fp32 residual add plus the
// bf16 copy the next layer's projection reads).
#include "common.cuh"

namespace kvs {
namespace proj {

constexpr int kWarps = 8;
#ifndef KVS_P1_CLUSTER
#define KVS_P1_CLUSTER 8
#endif
constexpr int kCluster = KVS_P1_CLUSTER;   // k-slices per 128 output columns
constexpr int kColsPerCluster = 16 * kWarps;   // 128
constexpr int kRowPad = 64;                    // bytes of padding per staged x row

__device__ __forceinline__ uint4 ldg_stream(const void *p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}
__device__ __forceinline__ void mma16816(float *c, uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 "
        "{%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, {%0, %1, %2, %3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::
                     : "memory");
}
__device__ __forceinline__ float ld_cluster_f32(uint32_t local_addr, uint32_t rank) {
    uint32_t remote;
    float v;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local_addr), "r"(rank));
    asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(remote) : "memory");
    return v;
}

// one 64-k iteration of a warp: rows g and g+8 of its 16 x 64 tile, two 32-k chunks each
struct WFrag {
    uint4 r0[2], r8[2];
};

template <int MT>
__global__ void __cluster_dims__(kCluster, 1, 1) __launch_bounds__(kWarps * 32)
    skinny_kernel(const __nv_bfloat16 *__restrict__ x, int m, const __nv_bfloat16 *__restrict__ w_p,
                  int n, int k, int accumulate, void *__restrict__ out,
                  __nv_bfloat16 *__restrict__ out_bf16) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int ks = k / kCluster;                        // k-slice of this CTA
    const int row_bytes = ks * 2 + kRowPad;
    uint8_t *xs = smem;                                 // [MT*8][ks] bf16, padded rows
    float *red = reinterpret_cast<float *>(smem);      // [MT*8][128] after the k loop (aliases xs)
    const uint32_t rank = cluster_rank();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    const int n0 = blockIdx.y * kColsPerCluster;
    const int k0 = (int)rank * ks;

    // stage x[:, k0:k0+ks] (rows >= m zero) as 16-byte pieces
    const int pieces = MT * 8 * (ks / 8);
    for (int p = threadIdx.x; p < pieces; p += blockDim.x) {
        const int r = p / (ks / 8), c = p - r * (ks / 8);
        uint4 v = make_uint4(0, 0, 0, 0);
        if (r < m) v = *reinterpret_cast<const uint4 *>(x + (size_t)r * k + k0 + c * 8);
        *reinterpret_cast<uint4 *>(xs + (size_t)r * row_bytes + c * 16) = v;
    }
    __syncthreads();

    // tile (n-group, k-block) at ((ng * k/64) + kb) * 1024 elements; lane (g, t) takes rows g
    // and g+8, k [8t, 8t+8) and [32+8t, 32+8t+8) of each tile
    const __nv_bfloat16 *wr0 = w_p + ((size_t)((n0 >> 4) + warp) * (k >> 6) + (k0 >> 6)) * 1024 +
                               g * 64 + 8 * t;
    const __nv_bfloat16 *wr8 = wr0 + 8 * 64;
    float acc[MT][4];
#pragma unroll
    for (int i = 0; i < MT; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;

    auto load = [&](WFrag &f, int kk) {
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            f.r0[c] = ldg_stream(wr0 + (kk >> 6) * 1024 + 32 * c);
            f.r8[c] = ldg_stream(wr8 + (kk >> 6) * 1024 + 32 * c);
        }
    };
    const uint8_t *xrow = xs + (size_t)g * row_bytes + 16 * t;
    auto compute = [&](const WFrag &f, int kk) {
#pragma unroll
        for (int c = 0; c < 2; ++c) {
#pragma unroll
            for (int rt = 0; rt < MT; ++rt) {
                const uint4 b = *reinterpret_cast<const uint4 *>(
                    xrow + (size_t)rt * 8 * row_bytes + (kk + 32 * c) * 2);
                mma16816(acc[rt], f.r0[c].x, f.r8[c].x, f.r0[c].y, f.r8[c].y, b.x, b.y);
                mma16816(acc[rt], f.r0[c].z, f.r8[c].z, f.r0[c].w, f.r8[c].w, b.z, b.w);
            }
        }
    };
    WFrag fa, fb;
    const int iters = ks / 64;
    load(fa, 0);
    for (int j = 0; j < iters; j += 2) {
        if (j + 1 < iters) load(fb, (j + 1) * 64);
        compute(fa, j * 64);
        if (j + 1 >= iters) break;
        if (j + 2 < iters) load(fa, (j + 2) * 64);
        compute(fb, (j + 1) * 64);
    }

    // partials: D[n][r] -> red[r][n_local] (the cross-cluster reads then run along n)
    constexpr int ldr = kColsPerCluster;
    __syncthreads();                                    // every warp is done with xs
#pragma unroll
    for (int rt = 0; rt < MT; ++rt) {
        const int r = rt * 8 + 2 * t, nl = warp * 16 + g;
        red[r * ldr + nl] = acc[rt][0];
        red[(r + 1) * ldr + nl] = acc[rt][1];
        red[r * ldr + nl + 8] = acc[rt][2];
        red[(r + 1) * ldr + nl + 8] = acc[rt][3];
    }
    cluster_sync();
    // rank c: columns [16c, 16c+16) of the cluster's 128, summed over the 8 slices in rank order
    const uint32_t red_addr = smem_u32(red);
    for (int e = threadIdx.x; e < 16 * m; e += blockDim.x) {
        const int r = e >> 4, nl = (int)rank * 16 + (e & 15);
        const uint32_t a = red_addr + (uint32_t)(r * ldr + nl) * 4u;
        float s = 0.f;
#pragma unroll
        for (int src = 0; src < kCluster; ++src) s += ld_cluster_f32(a, (uint32_t)src);
        const size_t o = (size_t)r * n + n0 + nl;
        if (accumulate) {
            float *of = reinterpret_cast<float *>(out);
            const float v = of[o] + s;
            of[o] = v;
            if (out_bf16 != nullptr) out_bf16[o] = __float2bfloat16_rn(v);
        } else {
            reinterpret_cast<__nv_bfloat16 *>(out)[o] = __float2bfloat16_rn(s);
        }
    }
    cluster_sync();    // the other ranks' reads of this CTA's partials are done
}

template <int MT>
static kvs_status launch(const void *x, int64_t m, const void *w_p, int64_t n, int64_t k,
                         int32_t accumulate, void *out, void *out_bf16, cudaStream_t s) {
    const int ks = (int)(k / kCluster);
    const size_t smem = (size_t)MT * 8 * (ks * 2 + kRowPad);    // the partials reuse it
    KVS_REQUIRE(smem <= 227 * 1024, KVS_ESHAPE, "skinny projection: k = %lld too large",
                (long long)k);
    cudaFuncSetAttribute(skinny_kernel<MT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    skinny_kernel<MT><<<dim3(kCluster, (unsigned)(n / kColsPerCluster)), kWarps * 32, smem, s>>>(
        static_cast<const __nv_bfloat16 *>(x), (int)m, static_cast<const __nv_bfloat16 *>(w_p),
        (int)n, (int)k, accumulate, out, static_cast<__nv_bfloat16 *>(out_bf16));
    KVS_CHECK_LAUNCH("kvs_proj_skinny");
    return KVS_OK;
}

}  // namespace proj
}  // namespace kvs

using namespace kvs;

extern "C" kvs_status kvs_proj_skinny(const void *x, int64_t m, const void *w_p, int64_t n,
                                      int64_t k, int32_t accumulate, void *out, void *out_bf16,
                                      kvs_stream_t stream) {
    KVS_REQUIRE(x != nullptr && w_p != nullptr && out != nullptr, KVS_EPARAM,
                "kvs_proj_skinny: null pointer");
    KVS_REQUIRE(m >= 1 && m <= 64, KVS_ESHAPE, "kvs_proj_skinny: m = %lld not in [1, 64]",
                (long long)m);
    KVS_REQUIRE(n > 0 && n % proj::kColsPerCluster == 0, KVS_ESHAPE,
                "kvs_proj_skinny: n = %lld not a multiple of 128", (long long)n);
    KVS_REQUIRE(k > 0 && k % (proj::kCluster * 64) == 0, KVS_ESHAPE,
                "kvs_proj_skinny: k = %lld not a multiple of 512", (long long)k);
    KVS_REQUIRE(((uintptr_t)x | (uintptr_t)w_p) % 16 == 0, KVS_EPARAM,
                "kvs_proj_skinny: x and w_p must be 16-byte aligned");
    KVS_REQUIRE(accumulate != 0 || out_bf16 == nullptr, KVS_EPARAM,
                "kvs_proj_skinny: out_bf16 only with accumulate");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (m <= 8) return proj::launch<1>(x, m, w_p, n, k, accumulate, out, out_bf16, s);
    if (m <= 16) return proj::launch<2>(x, m, w_p, n, k, accumulate, out, out_bf16, s);
    if (m <= 32) return proj::launch<4>(x, m, w_p, n, k, accumulate, out, out_bf16, s);
    return proj::launch<8>(x, m, w_p, n, k, accumulate, out, out_bf16, s);
}
