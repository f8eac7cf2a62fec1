// Shared helpers for the KVShare sm_100a kernels: status plumbing, bf16,
// warp primitives, and thin inline-PTX wrappers for mbarrier / TMA / tcgen05.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/kvshare.h"

namespace kvs {

// ---------------------------------------------------------------- status
void set_error(const char *fmt, ...);
kvs_status cuda_status(cudaError_t e, const char *where);

#define KVS_CHECK_LAUNCH(where)                                              \
    do {                                                                     \
        cudaError_t _e = cudaGetLastError();                                 \
        if (_e != cudaSuccess) return ::kvs::cuda_status(_e, where);         \
    } while (0)

#define KVS_REQUIRE(cond, code, ...)                                         \
    do {                                                                     \
        if (!(cond)) { ::kvs::set_error(__VA_ARGS__); return code; }         \
    } while (0)

constexpr int kNumSMs = 148;

// ---------------------------------------------------------------- math
__device__ __forceinline__ float bf2f(__nv_bfloat16 x) { return __bfloat162float(x); }
__device__ __forceinline__ __nv_bfloat16 f2bf(float x) { return __float2bfloat16_rn(x); }

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t *>(&v);
}

// Rotate-half RoPE on 8 dims [8c, 8c+8) of a head's first half (lo) and the
// paired dims of its second half (hi), coefficients in registers (two float4
// each).  Shared by the q/k scatter and the attention kernels' in-place Q
// rotation, so both produce the same bf16 bits.
__device__ __forceinline__ void rope8_reg(const uint4 &lo_in, const uint4 &hi_in, uint4 &lo_out,
                                          uint4 &hi_out, const float4 c0, const float4 c1,
                                          const float4 s0, const float4 s1) {
    const __nv_bfloat162 *x1 = reinterpret_cast<const __nv_bfloat162 *>(&lo_in);
    const __nv_bfloat162 *x2 = reinterpret_cast<const __nv_bfloat162 *>(&hi_in);
    uint32_t *o1 = reinterpret_cast<uint32_t *>(&lo_out);
    uint32_t *o2 = reinterpret_cast<uint32_t *>(&hi_out);
    const float cs[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
    const float sn[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const float2 a = __bfloat1622float2(x1[k]), b = __bfloat1622float2(x2[k]);
        // explicit fma/mul (no contraction choice left to the compiler)
        o1[k] = pack_bf16x2(__fmaf_rn(a.x, cs[2 * k], -__fmul_rn(b.x, sn[2 * k])),
                            __fmaf_rn(a.y, cs[2 * k + 1], -__fmul_rn(b.y, sn[2 * k + 1])));
        o2[k] = pack_bf16x2(__fmaf_rn(b.x, cs[2 * k], __fmul_rn(a.x, sn[2 * k])),
                            __fmaf_rn(b.y, cs[2 * k + 1], __fmul_rn(a.y, sn[2 * k + 1])));
    }
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

__device__ __forceinline__ float fast_exp2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Packed fp32 pairs (sm_100 FFMA2 / FADD2): two lanes of work per instruction,
// each rounded exactly like the scalar fmaf / fadd it replaces.
__device__ __forceinline__ void fma2(float &o0, float &o1, float a0, float a1, float b0, float b1,
                                     float c0, float c1) {
    asm("{\n.reg .b64 A, B, C, D;\n"
        "mov.b64 A, {%2, %3};\nmov.b64 B, {%4, %5};\nmov.b64 C, {%6, %7};\n"
        "fma.rn.f32x2 D, A, B, C;\nmov.b64 {%0, %1}, D;\n}"
        : "=f"(o0), "=f"(o1)
        : "f"(a0), "f"(a1), "f"(b0), "f"(b1), "f"(c0), "f"(c1));
}
__device__ __forceinline__ void add2(float &a0, float &a1, float b0, float b1) {
    asm("{\n.reg .b64 A, B, D;\n"
        "mov.b64 A, {%0, %1};\nmov.b64 B, {%2, %3};\n"
        "add.rn.f32x2 D, A, B;\nmov.b64 {%0, %1}, D;\n}"
        : "+f"(a0), "+f"(a1)
        : "f"(b0), "f"(b1));
}

// 2^x on the FMA pipe (no MUFU): round-to-nearest split x = j + f with the
// 1.5*2^23 magic add, cubic minimax for 2^f on [-0.5, 0.5] (relative error
// 7.5e-5, far below the bf16 rounding of P), exponent add for 2^j.  Used for
// a fraction of the softmax exponentials so MUFU and FMA pipes share the load.
__device__ __forceinline__ float exp2_poly(float x) {
    x = fmaxf(x, -126.f);
    const float t = x + 12582912.f;
    const float f = x - (t - 12582912.f);
    const float p = fmaf(fmaf(fmaf(0.0551716685f, f, 0.242611155f), f, 0.693260968f), f,
                         0.999928057f);
    return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}

// 32-byte global store (sm_100 STG.256): one full sector per thread.
__device__ __forceinline__ void st_global_v8(void *ptr, const uint32_t (&v)[8]) {
    asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(ptr), "r"(v[0]),
                 "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}

// exp2 of a pair on the FMA pipe with packed FADD2/FFMA2 (exp2_poly's
// rounding split and cubic, two lanes per instruction); the 2^j scaling is an
// integer add per lane.  Inputs clamped at -126.
__device__ __forceinline__ void exp2_poly2(float &y0, float &y1, float x0, float x1) {
    x0 = fmaxf(x0, -126.f);
    x1 = fmaxf(x1, -126.f);
    float t0, t1, r0, r1, f0, f1, p0, p1;
    fma2(t0, t1, x0, x1, 1.f, 1.f, 12582912.f, 12582912.f);       // x + 1.5*2^23
    fma2(r0, r1, t0, t1, 1.f, 1.f, -12582912.f, -12582912.f);     // round(x)
    fma2(f0, f1, r0, r1, -1.f, -1.f, x0, x1);                     // x - round(x)
    fma2(p0, p1, f0, f1, 0.0551716685f, 0.0551716685f, 0.242611155f, 0.242611155f);
    fma2(p0, p1, p0, p1, f0, f1, 0.693260968f, 0.693260968f);
    fma2(p0, p1, p0, p1, f0, f1, 0.999928057f, 0.999928057f);
    y0 = __int_as_float(__float_as_int(p0) + (__float_as_int(t0) << 23));
    y1 = __int_as_float(__float_as_int(p1) + (__float_as_int(t1) << 23));
}

// ---------------------------------------------------------------- smem / mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
// Watchdog: a wait that has not completed after ~2^24 suspended try_wait
// rounds (seconds) traps instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t addr = smem_u32(bar);
    uint32_t done = 0;
    for (uint32_t spin = 0;; ++spin) {
        asm volatile(
            "{\n"
            ".reg .pred P1;\n"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
            "selp.u32 %0, 1, 0, P1;\n"
            "}\n"
            : "=r"(done)
            : "r"(addr), "r"(parity)
            : "memory");
        if (done) return;
        if (spin > (1u << 24)) asm volatile("trap;");
    }
}

// Non-blocking phase test (for warps that poll several barriers).
__device__ __forceinline__ bool mbar_test(uint64_t *bar, uint32_t parity) {
    uint32_t done;
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
        "selp.u32 %0, 1, 0, P1;\n"
        "}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return done != 0;
}

__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---------------------------------------------------------------- TMA
__device__ __forceinline__ void tma_prefetch(const CUtensorMap *map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, uint64_t *bar,
                                            int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}
__device__ __forceinline__ void tma_load_4d(void *dst, const CUtensorMap *map, uint64_t *bar,
                                            int c0, int c1, int c2, int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2),
        "r"(c3)
        : "memory");
}

// ---------------------------------------------------------------- tcgen05
// Shared-memory matrix descriptor, SWIZZLE_128B, sm100 version bit set.
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr, uint32_t lbo_bytes,
                                                    uint32_t sbo_bytes) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;  // descriptor version (Blackwell)
    d |= (uint64_t)2 << 61;  // SWIZZLE_128B
    return d;
}

// Instruction descriptor: bf16 x bf16 -> f32, M x N, A K-major, B K- or MN-major.
__host__ __device__ constexpr uint32_t umma_idesc_bf16(int M, int N, bool b_mn_major) {
    return (1u << 4)          // D format f32
           | (1u << 7)        // A bf16
           | (1u << 10)       // B bf16
           | ((b_mn_major ? 1u : 0u) << 16) | ((uint32_t)(N >> 3) << 17) |
           ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void umma_bf16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                          uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

// A operand from tensor memory (TS form): a_tmem holds M rows x 16 K elements
// (bf16 packed two per 32-bit column, 8 columns); no output lanes disabled.
__device__ __forceinline__ void umma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                             uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, {%5, %6, %7, %8}, p;\n"
        "}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate), "r"(0u), "r"(0u), "r"(0u), "r"(0u));
}

__device__ __forceinline__ void umma_commit(uint64_t *bar) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void tmem_alloc(uint32_t *dst_smem, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(dst_smem)),
                 "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// 32 lanes x 32 columns of 32-bit: thread i of the warp gets lane (base+i), cols [c, c+32).
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float *v) {
    uint32_t *r = reinterpret_cast<uint32_t *>(v);
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
          "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
          "=r"(r[31])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float *v) {
    const uint32_t *r = reinterpret_cast<const uint32_t *>(v);
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
        "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
        "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),
        "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),
        "r"(r[29]), "r"(r[30]), "r"(r[31]));
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// ---------------------------------------------------------------- host TMA encode
// Driver entry point resolved through the runtime (no -lcuda needed).
bool encode_tmap(CUtensorMap *map, CUtensorMapDataType dtype, int rank, void *gaddr,
                 const uint64_t *dims, const uint64_t *strides_bytes /* rank-1 */,
                 const uint32_t *box, CUtensorMapSwizzle swz);

// The arena as a 4-D TMA tensor (dims: head_dim, kv head, page row, page x
// layer x K/V), box = 64 dims x 1 head x one page of rows, SWIZZLE_128B:
// one load brings half of a kv head's 128 dims for a page's 64 rows.
bool make_kv_map(CUtensorMap *m, const kvs_kv_arena *a);

// D3 fused decode-stage DHD (decode_dhd.cu), dispatched by kvs_dhd_decode_select.
size_t d3_counter_bytes();
size_t d3_fused_workspace(int32_t n_req, int32_t num_heads, int32_t max_ctx);
bool d3_fused_supported(const kvs_kv_arena *arena, int32_t n_req, int32_t num_heads,
                        int32_t n_extra);
kvs_status d3_fused_launch(const void *q_t, int32_t num_heads, const int32_t *ctx_len,
                           int32_t max_ctx, const float *dv_l1, uint8_t *eligible, int32_t layer,
                           const kvs_kv_arena *arena, const kvs_batch *batch, int32_t n_extra,
                           float softmax_scale, int32_t *chosen, int32_t *n_chosen, float *scores,
                           void *ws, cudaStream_t s);

}  // namespace kvs
