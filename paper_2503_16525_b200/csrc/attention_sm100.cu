// A1 selective-recompute attention and D1 DHD-alpha on sm_100a tensor cores.
//
// A1 (reference attention_forward inside _forward, model.py:110-129, 201, on
// the rows S a partial prefill computes - SURVEY.md A12): each CTA owns 128
// query rows of one head (scattered, ascending positions of one request) and
// streams that request's K/V pages from the paged arena with TMA
// (SWIZZLE_128B).  S = Q.K^T and O += P.V run as tcgen05.mma (M=128, N=128,
// K=16 steps) with S double-buffered and O resident in TMEM; 4 softmax warps
// (one query row per thread) apply the position-causal mask, an online
// softmax with lazy (threshold 2^8) O rescaling, and write P to shared
// memory in the canonical K-major SW128 layout.  Warp 4 = TMA producer,
// warp 5 = MMA issuer.
//
// D1 (reference v_impact_scores alpha, deviation.py:108-110): pass 1 is the
// same kernel without P.V (row log-sum-exp only); pass 2 swaps the operands -
// S^T = K_tile . Q_j^T with one KEY per TMEM lane - so the causal column sum
// sum_j exp(s_ji - lse_j) is a per-thread row reduction with no cross-thread
// traffic and no P store.
#include <algorithm>
#include <atomic>
#include <cstdlib>

#include "common.cuh"

namespace kvs {
namespace attn {

// Diagnostic timeline (KVS_ATTN_TRACE builds only): clock64 stamps of the
// first CTA's pipeline events, read back with kvs_attn_trace_dump().
#ifdef KVS_ATTN_TRACE
// one slot per (tag < 64, kb < 256): a plain store, no atomics, so tracing
// barely perturbs the pipeline it measures
__device__ long long g_trace[64 * 256];
#define TRACE(tag, kb)                                                              \
    do {                                                                            \
        if (blockIdx.y == 0 && blockIdx.x == 0 && (kb) < 256)                       \
            g_trace[(tag) * 256 + (kb)] = clock64();                                \
    } while (0)
#else
#define TRACE(tag, kb) do {} while (0)
#endif

constexpr int BM = 128, BN = 128, HD = 128;
constexpr int HALF_BYTES = 128 * 128;      // one [128 rows x 64 bf16] SW128 half tile
constexpr int TILE_BYTES = 2 * HALF_BYTES; // [128 rows x 128 bf16]
constexpr int NS = 2;                      // K/V stages
constexpr int kThreads = 192;
constexpr float kRescaleThreshold = 8.f;   // lazy rescale when max grows by > 2^8

struct Smem {
    uint64_t q_full;
    uint64_t k_full[NS], k_empty[NS], v_full[NS], v_empty[NS];
    uint64_t s_full[2], s_empty[2], p_full[2], pv_done[2];
    uint32_t tmem_base;
};

struct Params {
    const int32_t *row_pos;
    const int32_t *tile_req, *tile_row0, *tile_rows;
    const int32_t *kv_len;
    const int32_t *block_table;
    int32_t max_pages, page_size, num_layers, layer, num_heads, kv_heads, causal;
    float scale_log2;
    __nv_bfloat16 *out;
    float *lse;
    int64_t n_rows;
    // non-null: Q arrives un-rotated (straight from the QKV projection) and
    // the softmax warps rotate the tile in shared memory before the first
    // Q.K^T (fp32 [max_pos][64] cos/sin tables, the scatter's rotation)
    const float *q_cos, *q_sin;
    int32_t sched;        // persistent kernels: which ticket counter pair this launch uses
    // head selection of the persistent kernels: fwdp walks ppg head pairs per GQA
    // group (heads g*group + 2j, +1); fwd6p walks h_count heads k*h_stride + h_offset
    int32_t ppg, h_stride, h_offset, h_count;
};

// In-place rotation of row i of a TMA-loaded [128 x 128] SW128 Q tile: chunk
// c of the first half pairs with chunk c of the second half at the same
// swizzled offset.  Rows past the tile's end hold other rows or zeros and are
// rotated by position 0 (identity); their outputs are never stored.  The
// row's 64 cos + 64 sin coefficients are loaded into registers BEFORE the
// caller waits for the Q tile (load(), one L2 round trip hidden under the
// TMA), because shared stores through a generic pointer would otherwise keep
// the compiler from hoisting later chunks' table loads above them.
struct RopeRow {
    float4 c[16], s[16];
    __device__ __forceinline__ void load(int pos, const float *cos_t, const float *sin_t) {
        const float4 *c4 = reinterpret_cast<const float4 *>(cos_t + (size_t)pos * 64);
        const float4 *s4 = reinterpret_cast<const float4 *>(sin_t + (size_t)pos * 64);
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            c[k] = c4[k];
            s[k] = s4[k];
        }
    }
    __device__ __forceinline__ void apply(uint8_t *tile, int i) const {
        uint8_t *row = tile + i * 128;
        uint4 a[8], b[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            a[k] = *reinterpret_cast<const uint4 *>(row + ((k ^ (i & 7)) << 4));
            b[k] = *reinterpret_cast<const uint4 *>(row + HALF_BYTES + ((k ^ (i & 7)) << 4));
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            uint4 lo, hi;
            rope8_reg(a[k], b[k], lo, hi, c[2 * k], c[2 * k + 1], s[2 * k], s[2 * k + 1]);
            *reinterpret_cast<uint4 *>(row + ((k ^ (i & 7)) << 4)) = lo;
            *reinterpret_cast<uint4 *>(row + HALF_BYTES + ((k ^ (i & 7)) << 4)) = hi;
        }
    }
};

__device__ __forceinline__ uint32_t align1024(uint32_t a) { return (a + 1023u) & ~1023u; }

// D1 pass 1 (LSE, kPV = false): every kLsePoly-th exponential pair on the FMA
// pipe (exp2_poly2), 0 = all on MUFU.  1 in 4: 0.687 -> 0.643 ms (1 in 2 is
// slower, 0.784; A1 with its bf16 pack gets slower at any ratio)
#ifndef KVS_LSE_POLY
#define KVS_LSE_POLY 4
#endif
constexpr int kLsePoly = KVS_LSE_POLY;

template <bool kPV>
__global__ void __launch_bounds__(kThreads, kPV ? 1 : 2)
    fwd_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_kv,
               Params p) {
    extern __shared__ uint8_t dsmem[];
    __shared__ Smem sh;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tile = blockIdx.y, h = blockIdx.x;   // heads fastest: tiles in LPT order
    const int g = h / (p.num_heads / p.kv_heads);
    const int req = p.tile_req[tile], row0 = p.tile_row0[tile], nrows = p.tile_rows[tile];
    const int kmax = p.causal ? p.row_pos[row0 + nrows - 1] + 1 : p.kv_len[req];
    const int n_kb = (kmax + BN - 1) / BN;
    const int pages_needed = (kmax + p.page_size - 1) / p.page_size;

    const uint32_t base = align1024(smem_u32(dsmem));
    const uint32_t sQ = base;
    const uint32_t sK = sQ + TILE_BYTES;
    const uint32_t sV = sK + NS * TILE_BYTES;
    const uint32_t sP = sV + (kPV ? NS * TILE_BYTES : 0);
    uint8_t *gbase = dsmem + (base - smem_u32(dsmem));
    uint8_t *pP = gbase + (sP - base);

    if (threadIdx.x == 0) {
        mbar_init(&sh.q_full, 1);
        for (int i = 0; i < NS; ++i) {
            mbar_init(&sh.k_full[i], 1);
            mbar_init(&sh.k_empty[i], 1);
            mbar_init(&sh.v_full[i], 1);
            mbar_init(&sh.v_empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&sh.s_full[i], 1);
            mbar_init(&sh.s_empty[i], 128);
            mbar_init(&sh.p_full[i], 128);
            mbar_init(&sh.pv_done[i], 1);
        }
        fence_barrier_init();
    }
    // LSE-only launches (D1 pass 1) need S double-buffered and no O: 256
    // columns, so two CTAs share an SM (two softmax warps per SMSP)
    constexpr uint32_t kTmemCols = kPV ? 512 : 256;
    if (warp == 5) tmem_alloc(&sh.tmem_base, kTmemCols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = sh.tmem_base;
    const uint32_t tS[2] = {tmem, tmem + 128};
    const uint32_t tO = tmem + 256;

    if (warp == 4) {
        // ------------------------------------------------------------ TMA producer
        if (lane == 0) {
            tma_prefetch(&map_q);
            tma_prefetch(&map_kv);
            mbar_expect_tx(&sh.q_full, TILE_BYTES);
            for (int hf = 0; hf < 2; ++hf)
                tma_load_3d(gbase + (sQ - base) + hf * HALF_BYTES, &map_q, &sh.q_full, hf * 64, h,
                            row0);
            const int32_t *bt = p.block_table + (int64_t)req * p.max_pages;
            for (int kb = 0; kb < n_kb; ++kb) {
                const int st = kb % NS;
                const uint32_t ph = (uint32_t)((kb / NS) - 1) & 1u;
                int pg[2];
                for (int q = 0; q < 2; ++q) {
                    const int pi = 2 * kb + q;
                    pg[q] = bt[pi < pages_needed ? pi : 2 * kb];
                }
                if (kb >= NS) mbar_wait(&sh.k_empty[st], ph);
                mbar_expect_tx(&sh.k_full[st], TILE_BYTES);
                for (int q = 0; q < 2; ++q)
                    for (int hf = 0; hf < 2; ++hf)
                        tma_load_4d(gbase + (sK - base) + st * TILE_BYTES + hf * HALF_BYTES +
                                        q * (HALF_BYTES / 2),
                                    &map_kv, &sh.k_full[st], hf * 64, g, 0,
                                    (pg[q] * p.num_layers + p.layer) * 2 + 0);
                if (kPV) {
                    if (kb >= NS) mbar_wait(&sh.v_empty[st], ph);
                    mbar_expect_tx(&sh.v_full[st], TILE_BYTES);
                    for (int q = 0; q < 2; ++q)
                        for (int hf = 0; hf < 2; ++hf)
                            tma_load_4d(gbase + (sV - base) + st * TILE_BYTES + hf * HALF_BYTES +
                                            q * (HALF_BYTES / 2),
                                        &map_kv, &sh.v_full[st], hf * 64, g, 0,
                                        (pg[q] * p.num_layers + p.layer) * 2 + 1);
                }
            }
        }
    } else if (warp == 5) {
        // ------------------------------------------------------------ MMA issuer
        if (lane == 0) {
            const uint32_t idesc_qk = umma_idesc_bf16(BM, BN, false);
            const uint32_t idesc_pv = umma_idesc_bf16(BM, HD, true);
            mbar_wait(&sh.q_full, 0);
            auto issue_pv = [&](int j) {
                const int b = j & 1, st = j % NS;
                mbar_wait(&sh.p_full[b], (uint32_t)(j >> 1) & 1u);
                mbar_wait(&sh.v_full[st], (uint32_t)(j / NS) & 1u);
                tc_fence_after();
#pragma unroll
                for (int k = 0; k < BN / 16; ++k) {
                    const uint64_t da = umma_desc_sw128(sP + b * TILE_BYTES + (k >> 2) * HALF_BYTES +
                                                            (k & 3) * 32,
                                                        16, 1024);
                    const uint64_t db =
                        umma_desc_sw128(sV + st * TILE_BYTES + k * 2048, HALF_BYTES, 1024);
                    umma_bf16(tO, da, db, idesc_pv, (j > 0 || k > 0) ? 1u : 0u);
                }
                umma_commit(&sh.pv_done[b]);
                umma_commit(&sh.v_empty[st]);
            };
            for (int kb = 0; kb < n_kb; ++kb) {
                const int b = kb & 1, st = kb % NS;
                mbar_wait(&sh.k_full[st], (uint32_t)(kb / NS) & 1u);
                if (kb >= 2) mbar_wait(&sh.s_empty[b], (uint32_t)((kb >> 1) - 1) & 1u);
                tc_fence_after();
#pragma unroll
                for (int k = 0; k < HD / 16; ++k) {
                    const uint64_t da =
                        umma_desc_sw128(sQ + (k >> 2) * HALF_BYTES + (k & 3) * 32, 16, 1024);
                    const uint64_t db = umma_desc_sw128(
                        sK + st * TILE_BYTES + (k >> 2) * HALF_BYTES + (k & 3) * 32, 16, 1024);
                    umma_bf16(tS[b], da, db, idesc_qk, k > 0 ? 1u : 0u);
                }
                umma_commit(&sh.s_full[b]);
                umma_commit(&sh.k_empty[st]);
                if (kPV && kb >= 1) issue_pv(kb - 1);
            }
            if (kPV && n_kb >= 1) issue_pv(n_kb - 1);
        }
        __syncwarp();
    } else {
        // ------------------------------------------------------------ softmax warps 0-3
        const int i = threadIdx.x;  // row within tile == TMEM lane
        const bool valid = i < nrows;
        const int kend = !valid ? 0 : (p.causal ? p.row_pos[row0 + i] + 1 : kmax);
        const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
        float m = -INFINITY, l = 0.f;
        float s[BN];
        for (int kb = 0; kb < n_kb; ++kb) {
            const int b = kb & 1;
            mbar_wait(&sh.s_full[b], (uint32_t)(kb >> 1) & 1u);
            tc_fence_after();
#pragma unroll
            for (int c = 0; c < BN / 32; ++c) tmem_ld32(tS[b] + lane_off + c * 32, s + c * 32);
            tmem_ld_wait();
            tc_fence_before();
            mbar_arrive(&sh.s_empty[b]);
            const int kbase = kb * BN;
            if (!kPV && __all_sync(0xffffffffu, m != -INFINITY)) {
                // LSE pass (D1 pass 1): exponentials against the running max with
                // no max pass; only rows whose block sum exceeds 2^8 can hold a
                // term above 2^8 (fwdp's rule), and only their warps take the
                // exact path below
                if (kbase + BN > kend) {
#pragma unroll
                    for (int c = 0; c < BN; ++c) s[c] = (kbase + c < kend) ? s[c] : -INFINITY;
                }
                float ls[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) ls[j] = 0.f;
#pragma unroll
                for (int c = 0; c < BN; c += 2) {
                    float x0, x1, e0, e1;
                    fma2(x0, x1, s[c], s[c + 1], p.scale_log2, p.scale_log2, -m, -m);
                    if (kLsePoly > 0 && (c / 2) % (kLsePoly > 0 ? kLsePoly : 1) == kLsePoly - 1) {
                        exp2_poly2(e0, e1, x0, x1);
                    } else {
                        e0 = fast_exp2(x0);
                        e1 = fast_exp2(x1);
                    }
                    add2(ls[c & 7], ls[(c + 1) & 7], e0, e1);
                }
                const float bsum =
                    ((ls[0] + ls[1]) + (ls[2] + ls[3])) + ((ls[4] + ls[5]) + (ls[6] + ls[7]));
                if (!__any_sync(0xffffffffu, !(bsum <= 256.f))) {
                    l += bsum;
                    continue;
                }
            }
            // row max of the raw scores (scale > 0 commutes with max); the
            // position mask is only evaluated on blocks that cross this row's end
            float mx[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) mx[j] = -INFINITY;
            if (kbase + BN <= kend) {
#pragma unroll
                for (int c = 0; c < BN; ++c) mx[c & 7] = fmaxf(mx[c & 7], s[c]);
            } else {
#pragma unroll
                for (int c = 0; c < BN; ++c) {
                    s[c] = (kbase + c < kend) ? s[c] : -INFINITY;
                    mx[c & 7] = fmaxf(mx[c & 7], s[c]);
                }
            }
            const float mloc = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])),
                                     fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7]))) *
                               p.scale_log2;
            // lazy rescale: the decision is per row, but tcgen05.ld/st are
            // warp-collective, so the O pass runs for the whole warp whenever
            // any of its rows needs it (factor 1 on the others)
            const bool grow = mloc > m + kRescaleThreshold || (m == -INFINITY && mloc > -INFINITY);
            const bool touch_o = grow && kb >= 1 && m != -INFINITY;
            float factor = 1.f;
            if (grow) {
                factor = (m == -INFINITY) ? 0.f : fast_exp2(m - mloc);
                l *= factor;
                m = mloc;
            }
            if (kPV && __any_sync(0xffffffffu, touch_o)) {
                // O must be quiescent: wait for the previous P.V
                mbar_wait(&sh.pv_done[(kb - 1) & 1], (uint32_t)((kb - 1) >> 1) & 1u);
                tc_fence_after();
                const float f = touch_o ? factor : 1.f;
                float o[32];
#pragma unroll
                for (int c = 0; c < HD / 32; ++c) {
                    tmem_ld32(tO + lane_off + c * 32, o);
                    tmem_ld_wait();
#pragma unroll
                    for (int e = 0; e < 32; ++e) o[e] *= f;
                    tmem_st32(tO + lane_off + c * 32, o);
                }
                tmem_st_wait();
                tc_fence_before();
            }
            const float mu = (m == -INFINITY) ? 0.f : m;
            float ls[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) ls[j] = 0.f;
#pragma unroll
            for (int c = 0; c < BN; ++c) {
                const float e = fast_exp2(fmaf(s[c], p.scale_log2, -mu));
                s[c] = e;
                ls[c & 7] += e;
            }
            l += ((ls[0] + ls[1]) + (ls[2] + ls[3])) + ((ls[4] + ls[5]) + (ls[6] + ls[7]));
            if (kPV) {
                if (kb >= 2) mbar_wait(&sh.pv_done[b], (uint32_t)((kb - 2) >> 1) & 1u);
                uint8_t *prow = pP + b * TILE_BYTES + i * 128;
#pragma unroll
                for (int hf = 0; hf < 2; ++hf)
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        const float *x = s + hf * 64 + c * 8;
                        uint4 v;
                        v.x = pack_bf16x2(x[0], x[1]);
                        v.y = pack_bf16x2(x[2], x[3]);
                        v.z = pack_bf16x2(x[4], x[5]);
                        v.w = pack_bf16x2(x[6], x[7]);
                        *reinterpret_cast<uint4 *>(prow + hf * HALF_BYTES + ((c ^ (i & 7)) << 4)) = v;
                    }
                fence_proxy_async_smem();
                mbar_arrive(&sh.p_full[b]);
            }
        }
        const int64_t grow = (int64_t)row0 + i;
        if (kPV) {
            // every pv_done phase is waited on (PV(n_kb-2) was not, above)
            if (n_kb >= 2) mbar_wait(&sh.pv_done[n_kb & 1], (uint32_t)((n_kb - 2) >> 1) & 1u);
            if (n_kb >= 1) mbar_wait(&sh.pv_done[(n_kb - 1) & 1], (uint32_t)((n_kb - 1) >> 1) & 1u);
            tc_fence_after();
            const float inv = l > 0.f ? 1.f / l : 0.f;
            float o[32];
#pragma unroll
            for (int c = 0; c < HD / 32; ++c) {
                tmem_ld32(tO + lane_off + c * 32, o);
                tmem_ld_wait();
                if (valid && p.out != nullptr) {
                    uint4 *dst = reinterpret_cast<uint4 *>(
                        p.out + (grow * p.num_heads + h) * HD + c * 32);
#pragma unroll
                    for (int v = 0; v < 4; ++v) {
                        uint4 w;
                        w.x = pack_bf16x2(o[8 * v + 0] * inv, o[8 * v + 1] * inv);
                        w.y = pack_bf16x2(o[8 * v + 2] * inv, o[8 * v + 3] * inv);
                        w.z = pack_bf16x2(o[8 * v + 4] * inv, o[8 * v + 5] * inv);
                        w.w = pack_bf16x2(o[8 * v + 6] * inv, o[8 * v + 7] * inv);
                        dst[v] = w;
                    }
                }
            }
        }
        if (valid && p.lse != nullptr)
            p.lse[grow * p.num_heads + h] =
                (l > 0.f) ? (m + __log2f(l)) * 0.6931471805599453f : -INFINITY;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 5) {
        tc_fence_after();
        tmem_dealloc(tmem, kTmemCols);
    }
}

constexpr int kThreads2 = 384;   // fwd3: WG0, WG1 softmax; WG2 = TMA warp, MMA warp, 2 idle

// ------------------------------------------------------------------ A1, head pairs, P in TMEM
// CTA = 128 query rows x TWO query heads of the same GQA group: both heads
// read the same K/V tiles (one TMA stream, identical masks).  Warps 0-3 run
// head a's softmax, warps 4-7 head b's, warp 8 = TMA, warp 9 = MMA.  TMEM:
// S_a | S_b | O_a | O_b (128 columns each).  FA4 arrangement: the softmax
// writes P (bf16, two per column) back over its own S columns and O += P.V
// runs with A from tensor memory, so no P goes through shared memory and the
// K/V ring gets 5 slots.  The MMA warp issues
// PV_a(kb), QK_a(kb+1), PV_b(kb), QK_b(kb+1): in-order tcgen05 execution
// makes QK_t(kb+1) overwrite S/P only after PV_t(kb) has read P, and each
// head's softmax overlaps the other head's two MMAs.
constexpr int RING3 = 5;
#ifndef KVS_POLY_EVERY
#define KVS_POLY_EVERY 0
#endif
constexpr int kPolyEvery = KVS_POLY_EVERY;   // 1 in kPolyEvery exp2 pairs emulated (0: none)
#ifndef KVS_PINGPONG
#define KVS_PINGPONG 1
#endif
constexpr bool kPingPong = KVS_PINGPONG != 0;    // alternate the two heads' exp phases

struct Smem3 {
    uint64_t q_full, q_ready[2];
    uint64_t ring_full[RING3], ring_empty[RING3];
    uint64_t s_full[2], p_full[2], pv_done[2];
    uint32_t tmem_base;
};

__global__ void __launch_bounds__(kThreads2, 1)
    fwd3_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_kv,
                Params p) {
    extern __shared__ uint8_t dsmem[];
    __shared__ Smem3 sh;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tile = blockIdx.y, h0 = 2 * blockIdx.x;
    const int g = h0 / (p.num_heads / p.kv_heads);
    const int req = p.tile_req[tile], row0 = p.tile_row0[tile], nrows = p.tile_rows[tile];
    const int kmax = p.causal ? p.row_pos[row0 + nrows - 1] + 1 : p.kv_len[req];
    const int n_kb = (kmax + BN - 1) / BN;
    const int pages_needed = (kmax + p.page_size - 1) / p.page_size;

    const uint32_t base = align1024(smem_u32(dsmem));
    const uint32_t sQ = base;                          // 2 tiles
    const uint32_t sR = sQ + 2 * TILE_BYTES;           // RING3 tiles
    uint8_t *gbase = dsmem + (base - smem_u32(dsmem));

    if (threadIdx.x == 0) {
        mbar_init(&sh.q_full, 1);
        for (int i = 0; i < RING3; ++i) {
            mbar_init(&sh.ring_full[i], 1);
            mbar_init(&sh.ring_empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&sh.s_full[i], 1);
            mbar_init(&sh.p_full[i], 128);
            mbar_init(&sh.pv_done[i], 1);
            mbar_init(&sh.q_ready[i], 128);
        }
        fence_barrier_init();
    }
    if (warp == 9) tmem_alloc(&sh.tmem_base, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = sh.tmem_base;

    if (warp >= 8) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 88;");
        if (warp == 8 && lane == 0) {
            tma_prefetch(&map_q);
            tma_prefetch(&map_kv);
            mbar_expect_tx(&sh.q_full, 2 * TILE_BYTES);
            for (int t = 0; t < 2; ++t)
                for (int hf = 0; hf < 2; ++hf)
                    tma_load_3d(gbase + (sQ - base) + t * TILE_BYTES + hf * HALF_BYTES, &map_q,
                                &sh.q_full, hf * 64, h0 + t, row0);
            const int32_t *bt = p.block_table + (int64_t)req * p.max_pages;
            for (int it = 0; it < 2 * n_kb; ++it) {
                const int kb = it >> 1, kv = it & 1, slot = it % RING3;
                if (it >= RING3) mbar_wait(&sh.ring_empty[slot], (uint32_t)((it / RING3) - 1) & 1u);
                mbar_expect_tx(&sh.ring_full[slot], TILE_BYTES);
                for (int q = 0; q < 2; ++q) {
                    const int pi = 2 * kb + q;
                    const int pg = bt[pi < pages_needed ? pi : 2 * kb];
                    for (int hf = 0; hf < 2; ++hf)
                        tma_load_4d(gbase + (sR - base) + slot * TILE_BYTES + hf * HALF_BYTES +
                                        q * (HALF_BYTES / 2),
                                    &map_kv, &sh.ring_full[slot], hf * 64, g, 0,
                                    (pg * p.num_layers + p.layer) * 2 + kv);
                }
            }
        } else if (warp == 9 && lane == 0) {
            const uint32_t idesc_qk = umma_idesc_bf16(BM, BN, false);
            const uint32_t idesc_pv = umma_idesc_bf16(BM, HD, true);
            const bool qrope = p.q_cos != nullptr;
            if (!qrope) mbar_wait(&sh.q_full, 0);
            auto issue_qk = [&](int t, int kb) {
                const int slot = (2 * kb) % RING3;
#pragma unroll
                for (int k = 0; k < HD / 16; ++k) {
                    const uint64_t da = umma_desc_sw128(
                        sQ + t * TILE_BYTES + (k >> 2) * HALF_BYTES + (k & 3) * 32, 16, 1024);
                    const uint64_t db = umma_desc_sw128(
                        sR + slot * TILE_BYTES + (k >> 2) * HALF_BYTES + (k & 3) * 32, 16, 1024);
                    umma_bf16(tmem + 128 * t, da, db, idesc_qk, k > 0 ? 1u : 0u);
                }
                umma_commit(&sh.s_full[t]);
            };
            if (n_kb >= 1) {
                mbar_wait(&sh.ring_full[0], 0);
                tc_fence_after();
                for (int t = 0; t < 2; ++t) {
                    if (qrope) {                       // head t's Q rotated in place
                        mbar_wait(&sh.q_ready[t], 0);
                        tc_fence_after();
                    }
                    issue_qk(t, 0);
                }
                umma_commit(&sh.ring_empty[0]);
            }
            for (int kb = 0; kb < n_kb; ++kb) {
                const int itv = 2 * kb + 1, vslot = itv % RING3;
                const int itk = 2 * kb + 2, kslot = itk % RING3;
                const bool more = kb + 1 < n_kb;
                mbar_wait(&sh.ring_full[vslot], (uint32_t)(itv / RING3) & 1u);
                TRACE(10, kb);
                for (int t = 0; t < 2; ++t) {
                    mbar_wait(&sh.p_full[t], (uint32_t)kb & 1u);
                    TRACE(11 + t, kb);
                    tc_fence_after();
#pragma unroll
                    for (int k = 0; k < BN / 16; ++k) {
                        const uint64_t db = umma_desc_sw128(sR + vslot * TILE_BYTES + k * 2048,
                                                            HALF_BYTES, 1024);
                        umma_bf16_ts(tmem + 256 + 128 * t, tmem + 128 * t + 8 * k, db, idesc_pv,
                                     (kb > 0 || k > 0) ? 1u : 0u);
                    }
                    // O is read back once, after the last P.V: one pv_done phase
                    // per head (a phase nobody waits on is a synccheck error)
                    if (!more) umma_commit(&sh.pv_done[t]);
                    if (more) {
                        if (t == 0) mbar_wait(&sh.ring_full[kslot], (uint32_t)(itk / RING3) & 1u);
                        TRACE(13 + t, kb);
                        issue_qk(t, kb + 1);
                    }
                }
                umma_commit(&sh.ring_empty[vslot]);
                if (more) umma_commit(&sh.ring_empty[kslot]);
            }
        }
        __syncwarp();
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 208;");
        const int t = warp >> 2;                 // head of this warpgroup
        const int i = threadIdx.x & 127;         // row within tile == TMEM lane
        const bool valid = i < nrows;
        const int kend = !valid ? 0 : (p.causal ? p.row_pos[row0 + i] + 1 : kmax);
        const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
        const uint32_t tS = tmem + 128 * t + lane_off, tO = tmem + 256 + 128 * t + lane_off;
        if (p.q_cos != nullptr) {
            RopeRow rr;
            rr.load(valid ? p.row_pos[row0 + i] : 0, p.q_cos, p.q_sin);
            mbar_wait(&sh.q_full, 0);
            rr.apply(gbase + t * TILE_BYTES, i);
            fence_proxy_async_smem();                // generic writes -> tcgen05.mma reads
            mbar_arrive(&sh.q_ready[t]);
        }
        float m = -INFINITY, l = 0.f;
        float s[BN];
        for (int kb = 0; kb < n_kb; ++kb) {
            mbar_wait(&sh.s_full[t], (uint32_t)kb & 1u);
            if (i == 0) TRACE(20 + 10 * t, kb);
            tc_fence_after();
#pragma unroll
            for (int c = 0; c < BN / 32; ++c) tmem_ld32(tS + c * 32, s + c * 32);
            tmem_ld_wait();
            if (i == 0) TRACE(21 + 10 * t, kb);
            const int kbase = kb * BN;
            if (kbase + BN > kend) {                      // boundary block: position mask
#pragma unroll
                for (int c = 0; c < BN; ++c) s[c] = (kbase + c < kend) ? s[c] : -INFINITY;
            }
            float ls[8];
            // exponentials against mu, P (bf16) written over S; optionally the
            // block's row max is tracked in the same pass
            auto exp_pass = [&](float mu, bool track, float &bmax) {
                float mx[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    ls[j] = 0.f;
                    mx[j] = -INFINITY;
                }
#pragma unroll
                for (int hf = 0; hf < 2; ++hf) {
                    uint32_t pk[32];
#pragma unroll
                    for (int q = 0; q < 32; ++q) {
                        const float s0 = s[hf * 64 + 2 * q], s1 = s[hf * 64 + 2 * q + 1];
                        if (track) mx[q & 7] = fmaxf(mx[q & 7], fmaxf(s0, s1));
                        const float x0 = fmaf(s0, p.scale_log2, -mu);
                        const float x1 = fmaf(s1, p.scale_log2, -mu);
                        // every kPolyEvery-th pair on the FMA pipe, the rest on MUFU
                        const bool poly = kPolyEvery > 0 &&
                                          q % (kPolyEvery > 0 ? kPolyEvery : 1) == kPolyEvery - 1;
                        const float e0 = poly ? exp2_poly(x0) : fast_exp2(x0);
                        const float e1 = poly ? exp2_poly(x1) : fast_exp2(x1);
                        ls[(2 * q) & 7] += e0;
                        ls[(2 * q + 1) & 7] += e1;
                        pk[q] = pack_bf16x2(e0, e1);
                    }
                    tmem_st32(tS + hf * 32, reinterpret_cast<const float *>(pk));
                }
                if (track)
                    bmax = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])),
                                 fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
            };
            auto row_max = [&]() {
                float mx[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) mx[j] = -INFINITY;
#pragma unroll
                for (int c = 0; c < BN; ++c) mx[c & 7] = fmaxf(mx[c & 7], s[c]);
                return fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])),
                             fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
            };
            // lazy rescale: raise the running max m only when the block's max
            // exceeds it by > 2^8, rescaling O (warp-collective tcgen05 ops)
            auto rescale = [&](float mloc) {
                const bool grow = mloc > m + kRescaleThreshold || (m == -INFINITY && mloc > -INFINITY);
                const bool touch_o = grow && kb >= 1 && m != -INFINITY;
                float factor = 1.f;
                if (grow) {
                    factor = (m == -INFINITY) ? 0.f : fast_exp2(m - mloc);
                    l *= factor;
                    m = mloc;
                }
                if (__any_sync(0xffffffffu, touch_o)) {
                    // PV_t(kb-1) retired before QK_t(kb) (in-order), so O is quiescent
                    const float f = touch_o ? factor : 1.f;
                    float o[32];
#pragma unroll
                    for (int c = 0; c < HD / 32; ++c) {
                        tmem_ld32(tO + c * 32, o);
                        tmem_ld_wait();
#pragma unroll
                        for (int e = 0; e < 32; ++e) o[e] *= f;
                        tmem_st32(tO + c * 32, o);
                    }
                }
            };
            // ping-pong: the two heads' exponential phases alternate on the
            // shared MUFU pipe (16 lanes/clk/SM)
            if (kPingPong && (t == 1 || kb > 0))
                asm volatile("bar.sync %0, 256;" ::"r"(1 + t) : "memory");
            if (i == 0) TRACE(24 + 10 * t, kb);           // exp phase starts
            float bmax = -INFINITY;
            if (__all_sync(0xffffffffu, m != -INFINITY)) {
                // speculative pass against the running max (the common case:
                // no row's max grows by > 2^8), max tracked alongside; rows
                // that do grow make the warp redo the block with the new max
                exp_pass(m, true, bmax);
                if (__any_sync(0xffffffffu, bmax * p.scale_log2 > m + kRescaleThreshold)) {
                    rescale(bmax * p.scale_log2);
                    exp_pass(m, false, bmax);
                }
            } else {
                rescale(row_max() * p.scale_log2);
                exp_pass((m == -INFINITY) ? 0.f : m, false, bmax);
            }
            if (i == 0) TRACE(25 + 10 * t, kb);           // exp phase + P stores issued
            if (kPingPong) asm volatile("bar.arrive %0, 256;" ::"r"(2 - t) : "memory");
            l += ((ls[0] + ls[1]) + (ls[2] + ls[3])) + ((ls[4] + ls[5]) + (ls[6] + ls[7]));
            tmem_st_wait();
            if (i == 0) TRACE(22 + 10 * t, kb);
            tc_fence_before();
            mbar_arrive(&sh.p_full[t]);
        }
        if (kPingPong && t == 0 && n_kb >= 1) asm volatile("bar.sync 1, 256;" ::: "memory");
        const int64_t grow = (int64_t)row0 + i;
        if (n_kb >= 1) mbar_wait(&sh.pv_done[t], 0u);
        tc_fence_after();
        const float inv = l > 0.f ? 1.f / l : 0.f;
        float o[32];
#pragma unroll
        for (int c = 0; c < HD / 32; ++c) {
            tmem_ld32(tO + c * 32, o);
            tmem_ld_wait();
            if (valid) {
                uint4 *dst = reinterpret_cast<uint4 *>(p.out + (grow * p.num_heads + h0 + t) * HD +
                                                       c * 32);
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    uint4 w;
                    w.x = pack_bf16x2(o[8 * v + 0] * inv, o[8 * v + 1] * inv);
                    w.y = pack_bf16x2(o[8 * v + 2] * inv, o[8 * v + 3] * inv);
                    w.z = pack_bf16x2(o[8 * v + 4] * inv, o[8 * v + 5] * inv);
                    w.w = pack_bf16x2(o[8 * v + 6] * inv, o[8 * v + 7] * inv);
                    dst[v] = w;
                }
            }
        }
        if (valid && p.lse != nullptr)
            p.lse[grow * p.num_heads + h0 + t] =
                (l > 0.f) ? (m + __log2f(l)) * 0.6931471805599453f : -INFINITY;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 9) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// ------------------------------------------------------------------ A1, head pairs, persistent
// fwd3's pipeline in a persistent CTA (one per SM).  Work items (tile, head
// pair), in the host's tile order with head pairs fastest, are handed out by
// a global ticket: one-shot CTAs pay ~11 us of fixed cost each (metadata
// loads, Q/K TMA latency, the first Q.K^T, the O read-back and store,
// teardown) against ~1.9 us per 128-key block (tools/micro_attn_overhead.py),
// and a static round-robin walk loses that back to load imbalance.
//   * Warp 8 claims item k+1's ticket while item k streams, and publishes its
//     metadata and 128 row positions in a shared-memory slot (depth 3: the
//     softmax warps hold item k's slot until its epilogue), so no consumer
//     issues a dependent global load at an item boundary.
//   * Q_t(k+1) is loaded once the MMA warp commits q_empty[t] after item k's
//     last Q_t.K^T; with fused RoPE (p.q_cos) the softmax warps of head t
//     rotate it right after their last block of item k and arrive q_ready[t],
//     so Q.K^T(k+1, 0) runs under item k's epilogue.
//   * O_t(k) is read into registers and o_free[t] lets PV_t(k+1, 0) overwrite
//     it (accumulate = 0) before the normalised rows are stored.
// Barrier phases count blocks (s_full, p_full, ring) or items (q_*, pv_done,
// o_free, item slots) over the CTA's whole walk.
// exp-phase coupling of the two heads: 0 = none (both heads' softmax warps
// share each SMSP freely), 1 = strict ping-pong (one head's exp phase at a
// time), 2 = half offset (a head starts when the other is half done)
#ifndef KVS_PP_P
#define KVS_PP_P 0
#endif
constexpr int kPingPongP = KVS_PP_P;

struct ItemSlot {
    int w, req, row0, nrows, n_kb, kmax, h0, pad;
    int pos[BM];
};

struct SmemP {
    uint64_t q_full[2], q_empty[2], q_ready[2];
    uint64_t ring_full[RING3], ring_empty[RING3];
    uint64_t s_full[2], p_full[2], pv_done[2], o_free[2];
    uint64_t item_full[3], item_empty[3];
    uint32_t tmem_base;
    ItemSlot item[3];
};

// Ticket counters of the persistent kernels: pair [0] next ticket, [1] CTAs
// done; the last CTA of a launch zeroes its pair.  Each launch takes the next
// of kSchedSlots pairs round-robin (host side), so launches that overlap on
// different streams use different counters (up to kSchedSlots in flight).
constexpr int kSchedSlots = 64;
__device__ int g_fwdp_sched[kSchedSlots][2];

__global__ void __launch_bounds__(kThreads2, 1)
    fwdp_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_kv,
                Params p, int32_t n_items) {
    extern __shared__ uint8_t dsmem[];
    __shared__ SmemP sh;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int group = p.num_heads / p.kv_heads, pairs = p.kv_heads * p.ppg;
    const bool qrope = p.q_cos != nullptr;

    const uint32_t base = align1024(smem_u32(dsmem));
    const uint32_t sQ = base;                          // 2 tiles (one per head of the pair)
    const uint32_t sR = sQ + 2 * TILE_BYTES;           // RING3 tiles
    uint8_t *gbase = dsmem + (base - smem_u32(dsmem));

    if (threadIdx.x == 0) {
        for (int i = 0; i < RING3; ++i) {
            mbar_init(&sh.ring_full[i], 1);
            mbar_init(&sh.ring_empty[i], 1);
        }
        for (int t = 0; t < 2; ++t) {
            mbar_init(&sh.q_full[t], 1);
            mbar_init(&sh.q_empty[t], 1);
            mbar_init(&sh.q_ready[t], 128);
            mbar_init(&sh.s_full[t], 1);
            mbar_init(&sh.p_full[t], 128);
            mbar_init(&sh.pv_done[t], 1);
            mbar_init(&sh.o_free[t], 128);
        }
        for (int j = 0; j < 3; ++j) {
            mbar_init(&sh.item_full[j], 32);   // every producer lane releases its writes
            mbar_init(&sh.item_empty[j], 1 + 256);   // MMA lane + softmax threads
        }
        fence_barrier_init();
    }
    if (warp == 9) tmem_alloc(&sh.tmem_base, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = sh.tmem_base;

    if (warp >= 8) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 88;");
        if (warp == 8) {
            // ------------------------------------------------ tickets, item slots, TMA
            auto ticket = [&]() {
                int w = 0;
                if (lane == 0) w = atomicAdd(&g_fwdp_sched[p.sched][0], 1);
                return __shfl_sync(0xffffffffu, w, 0);
            };
            auto publish = [&](int k, int w) {       // item k = work item w -> slot k % 3
                const int s = k % 3;
                if (k >= 3) mbar_wait(&sh.item_empty[s], (uint32_t)((k / 3) - 1) & 1u);
                ItemSlot &it = sh.item[s];
                if (w < n_items) {
                    const int tile = w / pairs, pi = w - tile * pairs;
                    const int req = __ldg(p.tile_req + tile), row0 = __ldg(p.tile_row0 + tile);
                    const int nrows = __ldg(p.tile_rows + tile);
#pragma unroll
                    for (int r = lane; r < BM; r += 32)
                        it.pos[r] = r < nrows ? __ldg(p.row_pos + row0 + r) : 0;
                    if (lane == 0) {
                        const int kmax = p.causal ? __ldg(p.row_pos + row0 + nrows - 1) + 1
                                                  : __ldg(p.kv_len + req);
                        it.req = req;
                        it.row0 = row0;
                        it.nrows = nrows;
                        it.kmax = kmax;
                        it.n_kb = (kmax + BN - 1) / BN;
                        it.h0 = (pi / p.ppg) * group + 2 * (pi % p.ppg);   // both heads in one group
                    }
                }
                if (lane == 0) it.w = w;
                mbar_arrive(&sh.item_full[s]);
                __syncwarp();                        // lane 0's fields, for the warp's own reads
            };
            if (lane == 0) {
                tma_prefetch(&map_q);
                tma_prefetch(&map_kv);
            }
            int w = ticket();
            publish(0, w);
            int gb = 0, k = 0;
            while (w < n_items) {
                const ItemSlot &it = sh.item[k % 3];
                const int req = it.req, row0 = it.row0, n_kb = it.n_kb, kmax = it.kmax, h0 = it.h0;
                int wn = 0;
                {
                    const int g = h0 / group;
                    const int pages_needed = (kmax + p.page_size - 1) / p.page_size;
                    const int32_t *bt = p.block_table + (int64_t)req * p.max_pages;
                    for (int i2 = 0; i2 < 2 * n_kb; ++i2) {
                        if (lane == 0) {
                        if (i2 == 1) {
                            // Q after the first K tile: each waits on item k-1's last Q.K^T
                            for (int t = 0; t < 2; ++t) {
                                if (k >= 1) mbar_wait(&sh.q_empty[t], (uint32_t)(k - 1) & 1u);
                                TRACE(1 + t, k);
                                mbar_expect_tx(&sh.q_full[t], TILE_BYTES);
                                for (int hf = 0; hf < 2; ++hf)
                                    tma_load_3d(gbase + t * TILE_BYTES + hf * HALF_BYTES, &map_q,
                                                &sh.q_full[t], hf * 64, h0 + t, row0);
                            }
                        }
                        const int git = 2 * gb + i2, kb = i2 >> 1, kv = i2 & 1, slot = git % RING3;
                        if (git >= RING3)
                            mbar_wait(&sh.ring_empty[slot], (uint32_t)((git / RING3) - 1) & 1u);
                        mbar_expect_tx(&sh.ring_full[slot], TILE_BYTES);
                        for (int q = 0; q < 2; ++q) {
                            const int pi = 2 * kb + q;
                            const int pg = bt[pi < pages_needed ? pi : 2 * kb];
                            for (int hf = 0; hf < 2; ++hf)
                                tma_load_4d(gbase + (sR - base) + slot * TILE_BYTES +
                                                hf * HALF_BYTES + q * (HALF_BYTES / 2),
                                            &map_kv, &sh.ring_full[slot], hf * 64, g, 0,
                                            (pg * p.num_layers + p.layer) * 2 + kv);
                        }
                        }
                        if (i2 == 1) {
                            // item k's first K/V tiles and Q are in flight: claim and
                            // publish item k+1 (its ticket and metadata round trips
                            // overlap the ring waits that follow)
                            wn = ticket();
                            publish(k + 1, wn);
                        }
                    }
                }
                gb += n_kb;
                w = wn;
                ++k;
            }
            if (lane == 0 && atomicAdd(&g_fwdp_sched[p.sched][1], 1) == (int)gridDim.x - 1) {
                // every CTA has taken its last ticket: reset for the next launch
                atomicExch(&g_fwdp_sched[p.sched][0], 0);
                atomicExch(&g_fwdp_sched[p.sched][1], 0);
            }
        } else if (warp == 9 && lane == 0) {
            // ------------------------------------------------ MMA issuer
            const uint32_t idesc_qk = umma_idesc_bf16(BM, BN, false);
            const uint32_t idesc_pv = umma_idesc_bf16(BM, HD, true);
            auto issue_qk = [&](int t, int slot) {
#pragma unroll
                for (int k2 = 0; k2 < HD / 16; ++k2) {
                    const uint64_t da = umma_desc_sw128(
                        sQ + t * TILE_BYTES + (k2 >> 2) * HALF_BYTES + (k2 & 3) * 32, 16, 1024);
                    const uint64_t db = umma_desc_sw128(
                        sR + slot * TILE_BYTES + (k2 >> 2) * HALF_BYTES + (k2 & 3) * 32, 16, 1024);
                    umma_bf16(tmem + 128 * t, da, db, idesc_qk, k2 > 0 ? 1u : 0u);
                }
                umma_commit(&sh.s_full[t]);
            };
            int gb = 0;
            for (int k = 0;; ++k) {
                mbar_wait(&sh.item_full[k % 3], (uint32_t)(k / 3) & 1u);
                const int w = sh.item[k % 3].w, n_kb = sh.item[k % 3].n_kb;
                mbar_arrive(&sh.item_empty[k % 3]);
                if (w >= n_items) break;
                {
                    const int git = 2 * gb, slot = git % RING3;
                    mbar_wait(&sh.ring_full[slot], (uint32_t)(git / RING3) & 1u);
                    TRACE(3, k);
                    for (int t = 0; t < 2; ++t) {
                        mbar_wait(qrope ? &sh.q_ready[t] : &sh.q_full[t], (uint32_t)k & 1u);
                        TRACE(4 + t, k);
                        tc_fence_after();
                        issue_qk(t, slot);
                        if (n_kb == 1) umma_commit(&sh.q_empty[t]);
                    }
                    umma_commit(&sh.ring_empty[slot]);
                }
                for (int kb = 0; kb < n_kb; ++kb) {
                    const int gk = gb + kb;
                    const int itv = 2 * gk + 1, vslot = itv % RING3;
                    const int itk = 2 * gk + 2, kslot = itk % RING3;
                    const bool more = kb + 1 < n_kb;
                    mbar_wait(&sh.ring_full[vslot], (uint32_t)(itv / RING3) & 1u);
                    for (int t = 0; t < 2; ++t) {
                        mbar_wait(&sh.p_full[t], (uint32_t)gk & 1u);
                        // O_t of the previous item must have been read out
                        if (kb == 0 && k >= 1) mbar_wait(&sh.o_free[t], (uint32_t)(k - 1) & 1u);
                        TRACE(6 + t, gk);
                        tc_fence_after();
#pragma unroll
                        for (int k2 = 0; k2 < BN / 16; ++k2) {
                            const uint64_t db = umma_desc_sw128(sR + vslot * TILE_BYTES + k2 * 2048,
                                                                HALF_BYTES, 1024);
                            umma_bf16_ts(tmem + 256 + 128 * t, tmem + 128 * t + 8 * k2, db,
                                         idesc_pv, (kb > 0 || k2 > 0) ? 1u : 0u);
                        }
                        if (!more) umma_commit(&sh.pv_done[t]);
                        if (more) {
                            if (t == 0) mbar_wait(&sh.ring_full[kslot], (uint32_t)(itk / RING3) & 1u);
                            issue_qk(t, kslot);
                            if (kb + 2 == n_kb) umma_commit(&sh.q_empty[t]);
                        }
                    }
                    umma_commit(&sh.ring_empty[vslot]);
                    if (more) umma_commit(&sh.ring_empty[kslot]);
                }
                gb += n_kb;
            }
        }
        __syncwarp();
    } else {
        // ------------------------------------------------ softmax warpgroups
        asm volatile("setmaxnreg.inc.sync.aligned.u32 208;");
        const int t = warp >> 2;                 // head of this warpgroup
        const int i = threadIdx.x & 127;         // row within tile == TMEM lane
        const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
        const uint32_t tS = tmem + 128 * t + lane_off, tO = tmem + 256 + 128 * t + lane_off;
        // item kk's slot: published by warp 8, held until kk's epilogue has read it
        auto wait_item = [&](int kk) {
            mbar_wait(&sh.item_full[kk % 3], (uint32_t)(kk / 3) & 1u);
        };
        // rotate item kk's Q_t in place (row i's position) and release it to the MMA warp
        auto rope_q = [&](int kk) {
            RopeRow rr;
            rr.load(sh.item[kk % 3].pos[i], p.q_cos, p.q_sin);
            mbar_wait(&sh.q_full[t], (uint32_t)kk & 1u);
            rr.apply(gbase + t * TILE_BYTES, i);
            fence_proxy_async_smem();
            mbar_arrive(&sh.q_ready[t]);
        };
        int gb = 0, k = 0;
        wait_item(0);
        if (qrope && sh.item[0].w < n_items) rope_q(0);
        while (sh.item[k % 3].w < n_items) {
            const int slot = k % 3;
            const int n_kb = sh.item[slot].n_kb;
            const int kend = i >= sh.item[slot].nrows ? 0
                             : (p.causal ? sh.item[slot].pos[i] + 1 : sh.item[slot].kmax);
            float m = -INFINITY, l = 0.f;
            float s[BN];
            for (int kb = 0; kb < n_kb; ++kb) {
                const int gk = gb + kb;
                mbar_wait(&sh.s_full[t], (uint32_t)gk & 1u);
                if (i == 0) TRACE(20 + 10 * t, gk);
                tc_fence_after();
#pragma unroll
                for (int c = 0; c < BN / 32; ++c) tmem_ld32(tS + c * 32, s + c * 32);
                tmem_ld_wait();
                const int kbase = kb * BN;
                if (kbase + BN > kend) {
#pragma unroll
                    for (int c = 0; c < BN; ++c) s[c] = (kbase + c < kend) ? s[c] : -INFINITY;
                }
                float ls[8];
                auto exp_pass = [&](float mu, bool track, float &bmax, bool hook) {
                    float mx[8];
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        ls[j] = 0.f;
                        mx[j] = -INFINITY;
                    }
#pragma unroll
                    for (int hf = 0; hf < 2; ++hf) {
                        uint32_t pk[32];
#pragma unroll
                        for (int q = 0; q < 32; ++q) {
                            const float s0 = s[hf * 64 + 2 * q], s1 = s[hf * 64 + 2 * q + 1];
                            if (track) mx[q & 7] = fmaxf(mx[q & 7], fmaxf(s0, s1));
                            float x0, x1;
                            fma2(x0, x1, s0, s1, p.scale_log2, p.scale_log2, -mu, -mu);
                            // every kPolyEvery-th pair on the FMA pipe (0: all on MUFU)
                            const bool poly = kPolyEvery > 0 &&
                                              q % (kPolyEvery > 0 ? kPolyEvery : 1) == kPolyEvery - 1;
                            float e0, e1;
                            if (poly) {
                                exp2_poly2(e0, e1, x0, x1);
                            } else {
                                e0 = fast_exp2(x0);
                                e1 = fast_exp2(x1);
                            }
                            add2(ls[(2 * q) & 7], ls[(2 * q + 1) & 7], e0, e1);
                            pk[q] = pack_bf16x2(e0, e1);
                        }
                        tmem_st32(tS + hf * 32, reinterpret_cast<const float *>(pk));
                        if (kPingPongP == 2 && hook && hf == 0)
                            asm volatile("bar.arrive %0, 256;" ::"r"(2 - t) : "memory");
                    }
                    if (track)
                        bmax = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])),
                                     fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
                };
                auto row_max = [&]() {
                    float mx[8];
#pragma unroll
                    for (int j = 0; j < 8; ++j) mx[j] = -INFINITY;
#pragma unroll
                    for (int c = 0; c < BN; ++c) mx[c & 7] = fmaxf(mx[c & 7], s[c]);
                    return fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])),
                                 fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
                };
                auto rescale = [&](float mloc) {
                    const bool grow =
                        mloc > m + kRescaleThreshold || (m == -INFINITY && mloc > -INFINITY);
                    const bool touch_o = grow && kb >= 1 && m != -INFINITY;
                    float factor = 1.f;
                    if (grow) {
                        factor = (m == -INFINITY) ? 0.f : fast_exp2(m - mloc);
                        l *= factor;
                        m = mloc;
                    }
                    if (__any_sync(0xffffffffu, touch_o)) {
                        // PV_t(kb-1) retired before QK_t(kb) (in-order), so O is quiescent
                        const float f = touch_o ? factor : 1.f;
                        float o[32];
#pragma unroll
                        for (int c = 0; c < HD / 32; ++c) {
                            tmem_ld32(tO + c * 32, o);
                            tmem_ld_wait();
#pragma unroll
                            for (int e = 0; e < 32; ++e) o[e] *= f;
                            tmem_st32(tO + c * 32, o);
                        }
                    }
                };
                // ping-pong over the CTA's whole walk: head 1 waits on head 0's
                // exp phase of the same block, head 0 on head 1's previous one
                if (kPingPongP != 0 && (t == 1 || gk > 0))
                    asm volatile("bar.sync %0, 256;" ::"r"(1 + t) : "memory");
                float bmax = -INFINITY;
                if (__all_sync(0xffffffffu, m != -INFINITY)) {
                    // speculative pass against the running max with no per-element
                    // max tracking: a block term above 2^8 forces its sum above
                    // 2^8, so only rows whose block sum exceeds 2^8 (rare: terms
                    // are mostly < 1) take the exact max and maybe the redo
                    exp_pass(m, false, bmax, true);
                    const float bsum =
                        ((ls[0] + ls[1]) + (ls[2] + ls[3])) + ((ls[4] + ls[5]) + (ls[6] + ls[7]));
                    if (__any_sync(0xffffffffu, !(bsum <= 256.f))) {
                        bmax = row_max();
                        if (__any_sync(0xffffffffu, bmax * p.scale_log2 > m + kRescaleThreshold)) {
                            rescale(bmax * p.scale_log2);
                            exp_pass(m, false, bmax, false);
                        }
                    }
                } else {
                    rescale(row_max() * p.scale_log2);
                    exp_pass((m == -INFINITY) ? 0.f : m, false, bmax, true);
                }
                if (kPingPongP == 1) asm volatile("bar.arrive %0, 256;" ::"r"(2 - t) : "memory");
                l += ((ls[0] + ls[1]) + (ls[2] + ls[3])) + ((ls[4] + ls[5]) + (ls[6] + ls[7]));
                tmem_st_wait();
                tc_fence_before();
                mbar_arrive(&sh.p_full[t]);
                if (i == 0) TRACE(22 + 10 * t, gk);
            }
            // the next item's Q first (its Q.K^T then runs under this epilogue),
            // then O_t into registers, release it, normalise + store
            wait_item(k + 1);
            if (qrope && sh.item[(k + 1) % 3].w < n_items) rope_q(k + 1);
            if (i == 0) TRACE(25 + 10 * t, k);
            mbar_wait(&sh.pv_done[t], (uint32_t)k & 1u);
            if (i == 0) TRACE(26 + 10 * t, k);
            tc_fence_after();
            float o[HD];
#pragma unroll
            for (int c = 0; c < HD / 32; ++c) tmem_ld32(tO + c * 32, o + c * 32);
            tmem_ld_wait();
            tc_fence_before();
            mbar_arrive(&sh.o_free[t]);
            const int64_t grow = (int64_t)sh.item[slot].row0 + i;
            const int h = sh.item[slot].h0 + t;
            const bool valid = i < sh.item[slot].nrows;
            mbar_arrive(&sh.item_empty[slot]);
            const float inv = l > 0.f ? 1.f / l : 0.f;
            if (valid) {
                // 32-byte stores: each fills a whole sector of the row (16-byte
                // stores of rows 8 KB apart held the LSU ~1.5 us per item)
                __nv_bfloat16 *dst = p.out + (grow * p.num_heads + h) * HD;
#pragma unroll
                for (int v = 0; v < HD / 16; ++v) {
                    uint32_t wv[8];
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        wv[j] = pack_bf16x2(o[16 * v + 2 * j] * inv, o[16 * v + 2 * j + 1] * inv);
                    st_global_v8(dst + 16 * v, wv);
                }
                if (p.lse != nullptr)
                    p.lse[grow * p.num_heads + h] =
                        (l > 0.f) ? (m + __log2f(l)) * 0.6931471805599453f : -INFINITY;
            }
            if (i == 0) TRACE(27 + 10 * t, k);
            gb += n_kb;
            ++k;
        }
        mbar_arrive(&sh.item_empty[k % 3]);       // the terminal slot
        // consume head 1's last exp-phase arrival
        if (kPingPongP != 0 && t == 0 && gb >= 1) asm volatile("bar.sync 1, 256;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 9) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// ------------------------------------------------------------------ A1, one head, S double-buffered
// One query head per CTA; TMEM holds S0 | S1 | O (128 fp32 columns each).
// The softmax writes P (bf16) over the S buffer it read and O += P.V runs
// with A from tensor memory.  The MMA warp issues QK(kb+1) into the other S
// buffer right after PV(kb-1), so the next block's scores are computed while
// the softmax of this block runs and the softmax warps work back to back;
// in-order tcgen05 execution keeps QK(kb+2) behind PV(kb), which reads P(kb)
// from the same buffer.  Single softmax warpgroup: each warp owns its SMSP's
// MUFU.  K/V ring of 6 tiles (K(kb), V(kb), ...), 1 CTA per SM.
constexpr int RING6 = 6;
constexpr int kThreads6 = 192;

struct Smem6 {
    uint64_t q_full, q_ready;
    uint64_t ring_full[RING6], ring_empty[RING6];
    uint64_t s_full[2], p_full[2], pv_done[2];
    uint32_t tmem_base;
};

__global__ void __launch_bounds__(kThreads6, 1)
    fwd6_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_kv,
                Params p) {
    extern __shared__ uint8_t dsmem[];
    __shared__ Smem6 sh;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tile = blockIdx.y, h = blockIdx.x;
    const int g = h / (p.num_heads / p.kv_heads);
    const int req = p.tile_req[tile], row0 = p.tile_row0[tile], nrows = p.tile_rows[tile];
    const int kmax = p.causal ? p.row_pos[row0 + nrows - 1] + 1 : p.kv_len[req];
    const int n_kb = (kmax + BN - 1) / BN;
    const int pages_needed = (kmax + p.page_size - 1) / p.page_size;

    const uint32_t base = align1024(smem_u32(dsmem));
    const uint32_t sQ = base;                          // 1 tile
    const uint32_t sR = sQ + TILE_BYTES;               // RING6 tiles
    uint8_t *gbase = dsmem + (base - smem_u32(dsmem));

    if (threadIdx.x == 0) {
        mbar_init(&sh.q_full, 1);
        for (int i = 0; i < RING6; ++i) {
            mbar_init(&sh.ring_full[i], 1);
            mbar_init(&sh.ring_empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&sh.s_full[i], 1);
            mbar_init(&sh.p_full[i], 128);
            mbar_init(&sh.pv_done[i], 1);
        }
        mbar_init(&sh.q_ready, 128);
        fence_barrier_init();
    }
    if (warp == 5) tmem_alloc(&sh.tmem_base, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = sh.tmem_base;

    if (warp == 4) {
        if (lane == 0) {
            tma_prefetch(&map_q);
            tma_prefetch(&map_kv);
            mbar_expect_tx(&sh.q_full, TILE_BYTES);
            for (int hf = 0; hf < 2; ++hf)
                tma_load_3d(gbase + (sQ - base) + hf * HALF_BYTES, &map_q, &sh.q_full, hf * 64, h,
                            row0);
            const int32_t *bt = p.block_table + (int64_t)req * p.max_pages;
            for (int it = 0; it < 2 * n_kb; ++it) {
                const int kb = it >> 1, kv = it & 1, slot = it % RING6;
                if (it >= RING6) mbar_wait(&sh.ring_empty[slot], (uint32_t)((it / RING6) - 1) & 1u);
                mbar_expect_tx(&sh.ring_full[slot], TILE_BYTES);
                for (int q = 0; q < 2; ++q) {
                    const int pi = 2 * kb + q;
                    const int pg = bt[pi < pages_needed ? pi : 2 * kb];
                    for (int hf = 0; hf < 2; ++hf)
                        tma_load_4d(gbase + (sR - base) + slot * TILE_BYTES + hf * HALF_BYTES +
                                        q * (HALF_BYTES / 2),
                                    &map_kv, &sh.ring_full[slot], hf * 64, g, 0,
                                    (pg * p.num_layers + p.layer) * 2 + kv);
                }
            }
        }
    } else if (warp == 5) {
        if (lane == 0) {
            const uint32_t idesc_qk = umma_idesc_bf16(BM, BN, false);
            const uint32_t idesc_pv = umma_idesc_bf16(BM, HD, true);
            if (p.q_cos != nullptr) {                // Q rotated in place by the softmax warps
                mbar_wait(&sh.q_ready, 0);
                tc_fence_after();
            } else {
                mbar_wait(&sh.q_full, 0);
            }
            auto issue_qk = [&](int kb) {
                const int it = 2 * kb, slot = it % RING6, b = kb & 1;
                mbar_wait(&sh.ring_full[slot], (uint32_t)(it / RING6) & 1u);
                tc_fence_after();
#pragma unroll
                for (int k = 0; k < HD / 16; ++k) {
                    const uint64_t da =
                        umma_desc_sw128(sQ + (k >> 2) * HALF_BYTES + (k & 3) * 32, 16, 1024);
                    const uint64_t db = umma_desc_sw128(
                        sR + slot * TILE_BYTES + (k >> 2) * HALF_BYTES + (k & 3) * 32, 16, 1024);
                    umma_bf16(tmem + 128 * b, da, db, idesc_qk, k > 0 ? 1u : 0u);
                }
                umma_commit(&sh.s_full[b]);
                umma_commit(&sh.ring_empty[slot]);
            };
            auto issue_pv = [&](int kb) {
                const int it = 2 * kb + 1, slot = it % RING6, b = kb & 1;
                mbar_wait(&sh.p_full[b], (uint32_t)(kb >> 1) & 1u);
                mbar_wait(&sh.ring_full[slot], (uint32_t)(it / RING6) & 1u);
                tc_fence_after();
#pragma unroll
                for (int k = 0; k < BN / 16; ++k) {
                    const uint64_t db = umma_desc_sw128(sR + slot * TILE_BYTES + k * 2048,
                                                        HALF_BYTES, 1024);
                    umma_bf16_ts(tmem + 256, tmem + 128 * b + 8 * k, db, idesc_pv,
                                 (kb > 0 || k > 0) ? 1u : 0u);
                }
                umma_commit(&sh.pv_done[b]);
                umma_commit(&sh.ring_empty[slot]);
            };
            // QK(0), QK(1), PV(0), QK(2), PV(1), ...: QK(kb+1) runs under softmax(kb)
            if (n_kb >= 1) issue_qk(0);
            for (int kb = 0; kb < n_kb; ++kb) {
                if (kb + 1 < n_kb) issue_qk(kb + 1);
                issue_pv(kb);
            }
        }
        __syncwarp();
    } else {
        const int i = threadIdx.x;               // row within tile == TMEM lane
        const bool valid = i < nrows;
        const int kend = !valid ? 0 : (p.causal ? p.row_pos[row0 + i] + 1 : kmax);
        const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
        const uint32_t tO = tmem + 256 + lane_off;
        if (p.q_cos != nullptr) {
            RopeRow rr;
            rr.load(valid ? p.row_pos[row0 + i] : 0, p.q_cos, p.q_sin);
            mbar_wait(&sh.q_full, 0);
            rr.apply(gbase, i);
            fence_proxy_async_smem();
            mbar_arrive(&sh.q_ready);
        }
        float m = -INFINITY, l = 0.f;
        float s[BN];
        for (int kb = 0; kb < n_kb; ++kb) {
            const int b = kb & 1;
            const uint32_t tS = tmem + 128 * b + lane_off;
            mbar_wait(&sh.s_full[b], (uint32_t)(kb >> 1) & 1u);
            tc_fence_after();
#pragma unroll
            for (int c = 0; c < BN / 32; ++c) tmem_ld32(tS + c * 32, s + c * 32);
            tmem_ld_wait();
            const int kbase = kb * BN;
            if (kbase + BN > kend) {                      // boundary block: position mask
#pragma unroll
                for (int c = 0; c < BN; ++c) s[c] = (kbase + c < kend) ? s[c] : -INFINITY;
            }
            float ls[8];
            auto row_max = [&]() {
                float mx[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) mx[j] = -INFINITY;
#pragma unroll
                for (int c = 0; c < BN; ++c) mx[c & 7] = fmaxf(mx[c & 7], s[c]);
                return fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])),
                             fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
            };
            // lazy rescale (threshold 2^8); tcgen05.ld/st are warp-collective, so
            // the O pass runs for the whole warp when any of its rows needs it
            auto rescale = [&](float mloc) {
                const bool grow =
                    mloc > m + kRescaleThreshold || (m == -INFINITY && mloc > -INFINITY);
                const bool touch_o = grow && kb >= 1 && m != -INFINITY;
                float factor = 1.f;
                if (grow) {
                    factor = (m == -INFINITY) ? 0.f : fast_exp2(m - mloc);
                    l *= factor;
                    m = mloc;
                }
                if (__any_sync(0xffffffffu, touch_o)) {
                    // PV(kb-1) may still run: O is touched only after it retired
                    mbar_wait(&sh.pv_done[(kb - 1) & 1], (uint32_t)((kb - 1) >> 1) & 1u);
                    tc_fence_after();
                    const float f = touch_o ? factor : 1.f;
                    float o[32];
#pragma unroll
                    for (int c = 0; c < HD / 32; ++c) {
                        tmem_ld32(tO + c * 32, o);
                        tmem_ld_wait();
#pragma unroll
                        for (int e = 0; e < 32; ++e) o[e] *= f;
                        tmem_st32(tO + c * 32, o);
                    }
                    tmem_st_wait();
                }
            };
            auto exp_pass = [&](float mu) {
#pragma unroll
                for (int j = 0; j < 8; ++j) ls[j] = 0.f;
#pragma unroll
                for (int hf = 0; hf < 2; ++hf) {
                    uint32_t pk[32];
#pragma unroll
                    for (int q = 0; q < 32; ++q) {
                        float x0, x1;
                        fma2(x0, x1, s[hf * 64 + 2 * q], s[hf * 64 + 2 * q + 1], p.scale_log2,
                             p.scale_log2, -mu, -mu);
                        const float e0 = fast_exp2(x0), e1 = fast_exp2(x1);
                        add2(ls[(2 * q) & 7], ls[(2 * q + 1) & 7], e0, e1);
                        pk[q] = pack_bf16x2(e0, e1);
                    }
                    tmem_st32(tS + hf * 32, reinterpret_cast<const float *>(pk));
                }
            };
            if (__all_sync(0xffffffffu, m != -INFINITY)) {
                // speculative pass against the running max (fwdp's rule: only rows
                // whose block sum exceeds 2^8 can hold a term above 2^8)
                exp_pass(m);
                const float bsum =
                    ((ls[0] + ls[1]) + (ls[2] + ls[3])) + ((ls[4] + ls[5]) + (ls[6] + ls[7]));
                if (__any_sync(0xffffffffu, !(bsum <= 256.f))) {
                    const float bmax = row_max() * p.scale_log2;
                    if (__any_sync(0xffffffffu, bmax > m + kRescaleThreshold)) {
                        tmem_st_wait();                  // P stores done before S is rewritten
                        rescale(bmax);
                        exp_pass(m);
                    }
                }
            } else {
                rescale(row_max() * p.scale_log2);
                exp_pass((m == -INFINITY) ? 0.f : m);
            }
            l += ((ls[0] + ls[1]) + (ls[2] + ls[3])) + ((ls[4] + ls[5]) + (ls[6] + ls[7]));
            tmem_st_wait();
            tc_fence_before();
            mbar_arrive(&sh.p_full[b]);
            // consume PV(kb-1)'s phase (it ran under this block's softmax, so
            // the wait is free): every pv_done phase is waited on
            if (kb >= 1) mbar_wait(&sh.pv_done[(kb - 1) & 1], (uint32_t)((kb - 1) >> 1) & 1u);
        }
        const int64_t grow = (int64_t)row0 + i;
        if (n_kb >= 1) mbar_wait(&sh.pv_done[(n_kb - 1) & 1], (uint32_t)((n_kb - 1) >> 1) & 1u);
        tc_fence_after();
        const float inv = l > 0.f ? 1.f / l : 0.f;
        float o[32];
#pragma unroll
        for (int c = 0; c < HD / 32; ++c) {
            tmem_ld32(tO + c * 32, o);
            tmem_ld_wait();
            if (valid) {
                uint4 *dst = reinterpret_cast<uint4 *>(p.out + (grow * p.num_heads + h) * HD + c * 32);
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    uint4 w;
                    w.x = pack_bf16x2(o[8 * v + 0] * inv, o[8 * v + 1] * inv);
                    w.y = pack_bf16x2(o[8 * v + 2] * inv, o[8 * v + 3] * inv);
                    w.z = pack_bf16x2(o[8 * v + 4] * inv, o[8 * v + 5] * inv);
                    w.w = pack_bf16x2(o[8 * v + 6] * inv, o[8 * v + 7] * inv);
                    dst[v] = w;
                }
            }
        }
        if (valid && p.lse != nullptr)
            p.lse[grow * p.num_heads + h] =
                (l > 0.f) ? (m + __log2f(l)) * 0.6931471805599453f : -INFINITY;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 5) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// ------------------------------------------------------------------ A1, one head, persistent
// fwd6's pipeline (one query head, S double-buffered in TMEM, QK(kb+1) under
// softmax(kb)) in a persistent CTA walking (tile, head) items from a global
// ticket (fwdp's machinery: warp 4 publishes item metadata and row positions
// in shared memory).  Q is double-buffered (2 tiles + a 5-tile K/V ring), so
// item k+1's Q is loaded while item k runs and its first Q.K^T is issued
// right after item k's last one: the S-buffer alternation and the softmax
// warps run straight across item boundaries; only item k's epilogue (O read
// after its last P.V, then the stores) sits between softmax(k, last) and
// softmax(k+1, 0).  Barrier phases count blocks over the CTA's whole walk.
constexpr int RING6P = 5;

struct Smem6P {
    uint64_t q_full[2], q_empty[2];
    uint64_t ring_full[RING6P], ring_empty[RING6P];
    uint64_t s_full[2], p_full[2], pv_done[2];
    uint64_t item_full[3], item_empty[3];
    uint32_t tmem_base;
    ItemSlot item[3];
};

__device__ int g_fwd6p_sched[kSchedSlots][2];

__global__ void __launch_bounds__(kThreads6, 1)
    fwd6p_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_kv,
                 Params p, int32_t n_items) {
    extern __shared__ uint8_t dsmem[];
    __shared__ Smem6P sh;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int group = p.num_heads / p.kv_heads;

    const uint32_t base = align1024(smem_u32(dsmem));
    const uint32_t sQ = base;                          // 2 tiles: item k uses Q buffer k & 1
    const uint32_t sR = sQ + 2 * TILE_BYTES;           // RING6P tiles
    uint8_t *gbase = dsmem + (base - smem_u32(dsmem));

    if (threadIdx.x == 0) {
        for (int i = 0; i < RING6P; ++i) {
            mbar_init(&sh.ring_full[i], 1);
            mbar_init(&sh.ring_empty[i], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&sh.q_full[b], 1);
            mbar_init(&sh.q_empty[b], 1);
            mbar_init(&sh.s_full[b], 1);
            mbar_init(&sh.p_full[b], 128);
            mbar_init(&sh.pv_done[b], 1);
        }
        for (int j = 0; j < 3; ++j) {
            mbar_init(&sh.item_full[j], 32);   // every producer lane releases its writes
            mbar_init(&sh.item_empty[j], 1 + 128);   // MMA lane + softmax threads
        }
        fence_barrier_init();
    }
    if (warp == 5) tmem_alloc(&sh.tmem_base, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = sh.tmem_base;

    if (warp == 4) {
        // ------------------------------------------------ tickets, item slots, TMA
        auto ticket = [&]() {
            int w = 0;
            if (lane == 0) w = atomicAdd(&g_fwd6p_sched[p.sched][0], 1);
            return __shfl_sync(0xffffffffu, w, 0);
        };
        auto publish = [&](int k, int w) {           // item k = work item w -> slot k % 3
            const int s = k % 3;
            if (k >= 3) mbar_wait(&sh.item_empty[s], (uint32_t)((k / 3) - 1) & 1u);
            ItemSlot &it = sh.item[s];
            if (w < n_items) {
                const int tile = w / p.h_count;
                const int req = __ldg(p.tile_req + tile), row0 = __ldg(p.tile_row0 + tile);
                const int nrows = __ldg(p.tile_rows + tile);
#pragma unroll
                for (int r = lane; r < BM; r += 32)
                    it.pos[r] = r < nrows ? __ldg(p.row_pos + row0 + r) : 0;
                if (lane == 0) {
                    const int kmax = p.causal ? __ldg(p.row_pos + row0 + nrows - 1) + 1
                                              : __ldg(p.kv_len + req);
                    it.req = req;
                    it.row0 = row0;
                    it.nrows = nrows;
                    it.kmax = kmax;
                    it.n_kb = (kmax + BN - 1) / BN;
                    it.h0 = (w - tile * p.h_count) * p.h_stride + p.h_offset;
                }
            }
            if (lane == 0) it.w = w;
            mbar_arrive(&sh.item_full[s]);
            __syncwarp();                            // lane 0's fields, for the warp's own reads
        };
        auto load_q = [&](int k) {                   // item k's Q into buffer k & 1
            const ItemSlot &it = sh.item[k % 3];
            if (lane == 0 && it.w < n_items) {
                const int b = k & 1;
                if (k >= 2) mbar_wait(&sh.q_empty[b], (uint32_t)((k >> 1) - 1) & 1u);
                mbar_expect_tx(&sh.q_full[b], TILE_BYTES);
                for (int hf = 0; hf < 2; ++hf)
                    tma_load_3d(gbase + b * TILE_BYTES + hf * HALF_BYTES, &map_q, &sh.q_full[b],
                                hf * 64, it.h0, it.row0);
            }
        };
        if (lane == 0) {
            tma_prefetch(&map_q);
            tma_prefetch(&map_kv);
        }
        int w = ticket();
        publish(0, w);
        load_q(0);
        int gb = 0, k = 0;
        while (w < n_items) {
            const ItemSlot &it = sh.item[k % 3];
            const int req = it.req, n_kb = it.n_kb, kmax = it.kmax, gk = it.h0 / group;
            int wn = 0;
            const int pages_needed = (kmax + p.page_size - 1) / p.page_size;
            const int32_t *bt = p.block_table + (int64_t)req * p.max_pages;
            for (int i2 = 0; i2 < 2 * n_kb; ++i2) {
                if (lane == 0) {
                    const int git = 2 * gb + i2, kb = i2 >> 1, kv = i2 & 1, slot = git % RING6P;
                    if (git >= RING6P)
                        mbar_wait(&sh.ring_empty[slot], (uint32_t)((git / RING6P) - 1) & 1u);
                    mbar_expect_tx(&sh.ring_full[slot], TILE_BYTES);
                    for (int q = 0; q < 2; ++q) {
                        const int pi = 2 * kb + q;
                        const int pg = bt[pi < pages_needed ? pi : 2 * kb];
                        for (int hf = 0; hf < 2; ++hf)
                            tma_load_4d(gbase + (sR - base) + slot * TILE_BYTES + hf * HALF_BYTES +
                                            q * (HALF_BYTES / 2),
                                        &map_kv, &sh.ring_full[slot], hf * 64, gk, 0,
                                        (pg * p.num_layers + p.layer) * 2 + kv);
                    }
                }
                if (i2 == 1) {
                    // item k's first tiles are in flight: claim item k+1, publish
                    // it and start its Q load (buffer (k+1) & 1)
                    wn = ticket();
                    publish(k + 1, wn);
                    load_q(k + 1);
                }
            }
            gb += n_kb;
            w = wn;
            ++k;
        }
        if (lane == 0 && atomicAdd(&g_fwd6p_sched[p.sched][1], 1) == (int)gridDim.x - 1) {
            atomicExch(&g_fwd6p_sched[p.sched][0], 0);
            atomicExch(&g_fwd6p_sched[p.sched][1], 0);
        }
    } else if (warp == 5) {
        if (lane == 0) {
            // ------------------------------------------------ MMA issuer
            const uint32_t idesc_qk = umma_idesc_bf16(BM, BN, false);
            const uint32_t idesc_pv = umma_idesc_bf16(BM, HD, true);
            // QK of global block g (item buffer qb) into S[g & 1]
            auto issue_qk = [&](int g, int qb) {
                const int it = 2 * g, slot = it % RING6P;
                mbar_wait(&sh.ring_full[slot], (uint32_t)(it / RING6P) & 1u);
                tc_fence_after();
#pragma unroll
                for (int k2 = 0; k2 < HD / 16; ++k2) {
                    const uint64_t da = umma_desc_sw128(
                        sQ + qb * TILE_BYTES + (k2 >> 2) * HALF_BYTES + (k2 & 3) * 32, 16, 1024);
                    const uint64_t db = umma_desc_sw128(
                        sR + slot * TILE_BYTES + (k2 >> 2) * HALF_BYTES + (k2 & 3) * 32, 16, 1024);
                    umma_bf16(tmem + 128 * (g & 1), da, db, idesc_qk, k2 > 0 ? 1u : 0u);
                }
                umma_commit(&sh.s_full[g & 1]);
                umma_commit(&sh.ring_empty[slot]);
            };
            auto issue_pv = [&](int g, bool first) {
                const int it = 2 * g + 1, slot = it % RING6P, b = g & 1;
                mbar_wait(&sh.p_full[b], (uint32_t)(g >> 1) & 1u);
                mbar_wait(&sh.ring_full[slot], (uint32_t)(it / RING6P) & 1u);
                tc_fence_after();
#pragma unroll
                for (int k2 = 0; k2 < BN / 16; ++k2) {
                    const uint64_t db = umma_desc_sw128(sR + slot * TILE_BYTES + k2 * 2048,
                                                        HALF_BYTES, 1024);
                    umma_bf16_ts(tmem + 256, tmem + 128 * b + 8 * k2, db, idesc_pv,
                                 (!first || k2 > 0) ? 1u : 0u);
                }
                umma_commit(&sh.pv_done[b]);
                umma_commit(&sh.ring_empty[slot]);
            };
            int gb = 0;
            bool qk0_done = false;                   // item k's first QK issued under item k-1
            for (int k = 0;; ++k) {
                const int s = k % 3;
                mbar_wait(&sh.item_full[s], (uint32_t)(k / 3) & 1u);
                const int w = sh.item[s].w, n_kb = sh.item[s].n_kb;
                mbar_arrive(&sh.item_empty[s]);
                if (w >= n_items) break;
                if (!qk0_done) {
                    mbar_wait(&sh.q_full[k & 1], (uint32_t)(k >> 1) & 1u);
                    issue_qk(gb, k & 1);
                    if (n_kb == 1) umma_commit(&sh.q_empty[k & 1]);
                }
                qk0_done = false;
                for (int kb = 0; kb < n_kb; ++kb) {
                    const int g = gb + kb;
                    if (kb + 1 < n_kb) {
                        issue_qk(g + 1, k & 1);
                        if (kb + 2 == n_kb) umma_commit(&sh.q_empty[k & 1]);
                    } else {
                        // the next item's first QK goes ahead of this item's last P.V
                        const int s1 = (k + 1) % 3;
                        mbar_wait(&sh.item_full[s1], (uint32_t)((k + 1) / 3) & 1u);
                        if (sh.item[s1].w < n_items) {
                            mbar_wait(&sh.q_full[(k + 1) & 1], (uint32_t)((k + 1) >> 1) & 1u);
                            issue_qk(g + 1, (k + 1) & 1);
                            if (sh.item[s1].n_kb == 1) umma_commit(&sh.q_empty[(k + 1) & 1]);
                            qk0_done = true;
                        }
                    }
                    issue_pv(g, kb == 0);
                }
                gb += n_kb;
            }
        }
        __syncwarp();
    } else {
        // ------------------------------------------------ softmax warps 0-3
        const int i = threadIdx.x;               // row within tile == TMEM lane
        const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
        const uint32_t tO = tmem + 256 + lane_off;
        int gb = 0, k = 0;
        for (;; ++k) {
            const int slot = k % 3;
            mbar_wait(&sh.item_full[slot], (uint32_t)(k / 3) & 1u);
            if (sh.item[slot].w >= n_items) {
                mbar_arrive(&sh.item_empty[slot]);
                break;
            }
            const int n_kb = sh.item[slot].n_kb;
            const int kend = i >= sh.item[slot].nrows ? 0
                             : (p.causal ? sh.item[slot].pos[i] + 1 : sh.item[slot].kmax);
            float m = -INFINITY, l = 0.f;
            float s[BN];
            for (int kb = 0; kb < n_kb; ++kb) {
                const int g = gb + kb, b = g & 1;
                const uint32_t tS = tmem + 128 * b + lane_off;
                mbar_wait(&sh.s_full[b], (uint32_t)(g >> 1) & 1u);
                tc_fence_after();
#pragma unroll
                for (int c = 0; c < BN / 32; ++c) tmem_ld32(tS + c * 32, s + c * 32);
                tmem_ld_wait();
                const int kbase = kb * BN;
                if (kbase + BN > kend) {
#pragma unroll
                    for (int c = 0; c < BN; ++c) s[c] = (kbase + c < kend) ? s[c] : -INFINITY;
                }
                float ls[8];
                auto row_max = [&]() {
                    float mx[8];
#pragma unroll
                    for (int j = 0; j < 8; ++j) mx[j] = -INFINITY;
#pragma unroll
                    for (int c = 0; c < BN; ++c) mx[c & 7] = fmaxf(mx[c & 7], s[c]);
                    return fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])),
                                 fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
                };
                auto rescale = [&](float mloc) {
                    const bool grow =
                        mloc > m + kRescaleThreshold || (m == -INFINITY && mloc > -INFINITY);
                    const bool touch_o = grow && kb >= 1 && m != -INFINITY;
                    float factor = 1.f;
                    if (grow) {
                        factor = (m == -INFINITY) ? 0.f : fast_exp2(m - mloc);
                        l *= factor;
                        m = mloc;
                    }
                    if (__any_sync(0xffffffffu, touch_o)) {
                        // PV(g-1) may still run: O is touched only after it retired
                        mbar_wait(&sh.pv_done[(g - 1) & 1], (uint32_t)((g - 1) >> 1) & 1u);
                        tc_fence_after();
                        const float f = touch_o ? factor : 1.f;
                        float o[32];
#pragma unroll
                        for (int c = 0; c < HD / 32; ++c) {
                            tmem_ld32(tO + c * 32, o);
                            tmem_ld_wait();
#pragma unroll
                            for (int e = 0; e < 32; ++e) o[e] *= f;
                            tmem_st32(tO + c * 32, o);
                        }
                        tmem_st_wait();
                    }
                };
                auto exp_pass = [&](float mu) {
#pragma unroll
                    for (int j = 0; j < 8; ++j) ls[j] = 0.f;
#pragma unroll
                    for (int hf = 0; hf < 2; ++hf) {
                        uint32_t pk[32];
#pragma unroll
                        for (int q = 0; q < 32; ++q) {
                            float x0, x1;
                            fma2(x0, x1, s[hf * 64 + 2 * q], s[hf * 64 + 2 * q + 1], p.scale_log2,
                                 p.scale_log2, -mu, -mu);
                            const float e0 = fast_exp2(x0), e1 = fast_exp2(x1);
                            add2(ls[(2 * q) & 7], ls[(2 * q + 1) & 7], e0, e1);
                            pk[q] = pack_bf16x2(e0, e1);
                        }
                        tmem_st32(tS + hf * 32, reinterpret_cast<const float *>(pk));
                    }
                };
                if (__all_sync(0xffffffffu, m != -INFINITY)) {
                    exp_pass(m);
                    const float bsum =
                        ((ls[0] + ls[1]) + (ls[2] + ls[3])) + ((ls[4] + ls[5]) + (ls[6] + ls[7]));
                    if (__any_sync(0xffffffffu, !(bsum <= 256.f))) {
                        const float bmax = row_max() * p.scale_log2;
                        if (__any_sync(0xffffffffu, bmax > m + kRescaleThreshold)) {
                            tmem_st_wait();
                            rescale(bmax);
                            exp_pass(m);
                        }
                    }
                } else {
                    rescale(row_max() * p.scale_log2);
                    exp_pass((m == -INFINITY) ? 0.f : m);
                }
                l += ((ls[0] + ls[1]) + (ls[2] + ls[3])) + ((ls[4] + ls[5]) + (ls[6] + ls[7]));
                tmem_st_wait();
                tc_fence_before();
                mbar_arrive(&sh.p_full[b]);
                // consume PV(g-1)'s phase (free: it ran under this block's softmax)
                if (kb >= 1) mbar_wait(&sh.pv_done[(g - 1) & 1], (uint32_t)((g - 1) >> 1) & 1u);
            }
            // epilogue: O after the item's last P.V, read before the next item's
            // first P.V (issued only after this thread's next p_full arrival)
            const int gl = gb + n_kb - 1;
            mbar_wait(&sh.pv_done[gl & 1], (uint32_t)(gl >> 1) & 1u);
            tc_fence_after();
            float o[HD];
#pragma unroll
            for (int c = 0; c < HD / 32; ++c) tmem_ld32(tO + c * 32, o + c * 32);
            tmem_ld_wait();
            tc_fence_before();
            const int64_t grow = (int64_t)sh.item[slot].row0 + i;
            const int h = sh.item[slot].h0;
            const bool valid = i < sh.item[slot].nrows;
            mbar_arrive(&sh.item_empty[slot]);
            const float inv = l > 0.f ? 1.f / l : 0.f;
            if (valid) {
                __nv_bfloat16 *dst = p.out + (grow * p.num_heads + h) * HD;
#pragma unroll
                for (int v = 0; v < HD / 16; ++v) {
                    uint32_t wv[8];
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        wv[j] = pack_bf16x2(o[16 * v + 2 * j] * inv, o[16 * v + 2 * j + 1] * inv);
                    st_global_v8(dst + 16 * v, wv);
                }
                if (p.lse != nullptr)
                    p.lse[grow * p.num_heads + h] =
                        (l > 0.f) ? (m + __log2f(l)) * 0.6931471805599453f : -INFINITY;
            }
            gb += n_kb;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 5) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// ------------------------------------------------------------------ D1 pass 2
// D1's exponentials have no bf16 pack and two softmax warps per SMSP keep the
// MUFU pipe busy, so half of the colsum / LSE-pass pairs go to the FMA pipe
// (exp2_poly2): colsum 0.979 -> 0.913 ms (tools/micro_alpha.py)
#ifndef KVS_D1_POLY
#define KVS_D1_POLY 2
#endif
#ifndef KVS_D1_POLY_NUM
#define KVS_D1_POLY_NUM 1
#endif
constexpr int kD1Poly = KVS_D1_POLY, kD1PolyNum = KVS_D1_POLY_NUM;
// CTA = (key tile kt of request r, kv head g).  Loops over the group's query
// heads and the query tiles that can see the keys; S^T lands with one key per
// TMEM lane, so each softmax thread accumulates its key's column sum.
struct ColParams {
    const int64_t *req_off;
    const int32_t *row_pos;
    const int32_t *tile_req, *tile_row0;  // key tiles == the probe's row tiles
    const float *lse;                   // [n_total][H] natural log
    const int32_t *block_table;
    int32_t max_pages, page_size, num_layers, layer, num_heads, kv_heads, causal;
    float scale_log2;
    float *alpha_part;                  // [n_total][kv_heads]
};

__global__ void __launch_bounds__(kThreads, 2)
    colsum_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_kv,
                  ColParams p) {
    extern __shared__ uint8_t dsmem[];
    __shared__ Smem sh;
    __shared__ float s_lse[2][BM];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // key tiles fastest: the CTAs of one kv group sweep a few requests at a
    // time, so those requests' query tiles are re-read from L2, not DRAM
    const int tile = blockIdx.x, g = blockIdx.y;
    const int hq = p.num_heads / p.kv_heads;
    const int req = p.tile_req[tile], k0 = p.row_pos[p.tile_row0[tile]];
    const int64_t s0 = p.req_off[req];
    const int n = (int)(p.req_off[req + 1] - s0);
    const int q_first = p.causal ? (k0 / BM) : 0;         // first query tile that sees the keys
    const int n_qt = (n + BM - 1) / BM - q_first;
    const int n_it = hq * n_qt;                            // (head, query tile) iterations

    const uint32_t base = align1024(smem_u32(dsmem));
    const uint32_t sK = base;                  // A operand: the key tile (resident)
    const uint32_t sQ = sK + TILE_BYTES;       // B operand stages: query tiles
    uint8_t *gbase = dsmem + (base - smem_u32(dsmem));

    if (threadIdx.x == 0) {
        mbar_init(&sh.q_full, 1);
        for (int i = 0; i < NS; ++i) {
            mbar_init(&sh.k_full[i], 1);
            mbar_init(&sh.k_empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&sh.s_full[i], 1);
            mbar_init(&sh.s_empty[i], 128);
        }
        fence_barrier_init();
    }
    if (warp == 5) tmem_alloc(&sh.tmem_base, 256);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = sh.tmem_base;
    const uint32_t tS[2] = {tmem, tmem + 128};

    if (warp == 4) {
        if (lane == 0) {
            tma_prefetch(&map_q);
            tma_prefetch(&map_kv);
            const int32_t *bt = p.block_table + (int64_t)req * p.max_pages;
            const int pages = (n + p.page_size - 1) / p.page_size;
            mbar_expect_tx(&sh.q_full, TILE_BYTES);  // key tile rides on q_full
            for (int q = 0; q < 2; ++q) {
                const int pi = k0 / p.page_size + q;
                const int pg = bt[pi < pages ? pi : k0 / p.page_size];
                for (int hf = 0; hf < 2; ++hf)
                    tma_load_4d(gbase + (sK - base) + hf * HALF_BYTES + q * (HALF_BYTES / 2),
                                &map_kv, &sh.q_full, hf * 64, g, 0,
                                (pg * p.num_layers + p.layer) * 2 + 0);
            }
            for (int it = 0; it < n_it; ++it) {
                const int st = it % NS;
                const int hh = it / n_qt, qt = q_first + it % n_qt;
                if (it >= NS) mbar_wait(&sh.k_empty[st], (uint32_t)((it / NS) - 1) & 1u);
                mbar_expect_tx(&sh.k_full[st], TILE_BYTES);
                for (int hf = 0; hf < 2; ++hf)
                    tma_load_3d(gbase + (sQ - base) + st * TILE_BYTES + hf * HALF_BYTES, &map_q,
                                &sh.k_full[st], hf * 64, g * hq + hh, (int)(s0 + qt * BM));
            }
        }
    } else if (warp == 5) {
        if (lane == 0) {
            const uint32_t idesc = umma_idesc_bf16(BM, BN, false);
            mbar_wait(&sh.q_full, 0);
            for (int it = 0; it < n_it; ++it) {
                const int b = it & 1, st = it % NS;
                mbar_wait(&sh.k_full[st], (uint32_t)(it / NS) & 1u);
                if (it >= 2) mbar_wait(&sh.s_empty[b], (uint32_t)((it >> 1) - 1) & 1u);
                tc_fence_after();
#pragma unroll
                for (int k = 0; k < HD / 16; ++k) {
                    const uint64_t da =
                        umma_desc_sw128(sK + (k >> 2) * HALF_BYTES + (k & 3) * 32, 16, 1024);
                    const uint64_t db = umma_desc_sw128(
                        sQ + st * TILE_BYTES + (k >> 2) * HALF_BYTES + (k & 3) * 32, 16, 1024);
                    umma_bf16(tS[b], da, db, idesc, k > 0 ? 1u : 0u);
                }
                umma_commit(&sh.s_full[b]);
                umma_commit(&sh.k_empty[st]);
            }
        }
        __syncwarp();
    } else {
        const int i = threadIdx.x;               // key within tile == TMEM lane
        const int kpos = k0 + i;
        const bool kvalid = kpos < n;
        const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
        float acc = 0.f;
        float s[BN];
        // the query LSEs of iteration it+1 are loaded while iteration it
        // computes (a load issued right before the barrier below would expose
        // its L2 latency on every iteration)
        auto lse_of = [&](int it) {
            const int hh = it / n_qt, qt = q_first + it % n_qt;
            const int qrow = qt * BM + i;
            return qrow < n ? __ldg(p.lse + (s0 + qrow) * p.num_heads + g * hq + hh) : INFINITY;
        };
        float lse_next = n_it > 0 ? lse_of(0) : 0.f;
        for (int it = 0; it < n_it; ++it) {
            const int b = it & 1;
            const int qt = q_first + it % n_qt;
            // stage this iteration's query LSEs (log2 units) in shared memory
            s_lse[b][i] = lse_next * 1.4426950408889634f;
            if (it + 1 < n_it) lse_next = lse_of(it + 1);
            asm volatile("bar.sync 1, 128;" ::: "memory");
            mbar_wait(&sh.s_full[b], (uint32_t)(it >> 1) & 1u);
            tc_fence_after();
#pragma unroll
            for (int c = 0; c < BN / 32; ++c) tmem_ld32(tS[b] + lane_off + c * 32, s + c * 32);
            tmem_ld_wait();
            tc_fence_before();
            mbar_arrive(&sh.s_empty[b]);
            const int qbase = qt * BM;
            float ps[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) ps[j] = 0.f;
            if (!p.causal || qbase >= k0 + BM - 1) {
                // every query of this tile sees every key of the key tile
#pragma unroll
                for (int c = 0; c < BN; c += 2) {
                    float x0, x1, e0, e1;
                    fma2(x0, x1, s[c], s[c + 1], p.scale_log2, p.scale_log2, -s_lse[b][c],
                         -s_lse[b][c + 1]);
                    // every KVS_D1_POLY-th pair of exponentials on the FMA pipe
                    if (kD1Poly > 0 && (c / 2) % (kD1Poly > 0 ? kD1Poly : 1) >= kD1Poly - kD1PolyNum) {
                        exp2_poly2(e0, e1, x0, x1);
                    } else {
                        e0 = fast_exp2(x0);
                        e1 = fast_exp2(x1);
                    }
                    add2(ps[c & 7], ps[(c + 1) & 7], e0, e1);
                }
            } else {
#pragma unroll
                for (int c = 0; c < BN; c += 2) {
                    float x0, x1;
                    fma2(x0, x1, s[c], s[c + 1], p.scale_log2, p.scale_log2, -s_lse[b][c],
                         -s_lse[b][c + 1]);
                    const float e0 = fast_exp2(x0), e1 = fast_exp2(x1);
                    add2(ps[c & 7], ps[(c + 1) & 7], (qbase + c >= kpos) ? e0 : 0.f,
                         (qbase + c + 1 >= kpos) ? e1 : 0.f);
                }
            }
            const float part = ((ps[0] + ps[1]) + (ps[2] + ps[3])) + ((ps[4] + ps[5]) + (ps[6] + ps[7]));
            acc += part;
        }
        if (kvalid) p.alpha_part[(s0 + kpos) * p.kv_heads + g] = acc;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 5) {
        tc_fence_after();
        tmem_dealloc(tmem, 256);
    }
}

__global__ void alpha_reduce_kernel(const float *__restrict__ part, int64_t n, int32_t G, int32_t H,
                                    float *__restrict__ alpha) {
    // D2 (launched programmatically dependent) may start its prologue now;
    // it waits for this grid's completion before it reads alpha
    asm volatile("griddepcontrol.launch_dependents;");
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
         t += (int64_t)gridDim.x * blockDim.x) {
        float s = 0.f;
        for (int g = 0; g < G; ++g) s += part[t * G + g];
        alpha[t] = s / (float)H;
    }
}

}  // namespace attn

// q: [n_rows][row_stride] bf16 whose first H*D elements are the query heads
// (row_stride = H*D for a dense q, (H+2G)*D for rows of the QKV projection)
static bool make_q_map(CUtensorMap *m, const void *q, int64_t n_rows, int H, int D,
                       int64_t row_stride = 0) {
    if (row_stride == 0) row_stride = (int64_t)H * D;
    uint64_t dims[3] = {(uint64_t)D, (uint64_t)H, (uint64_t)n_rows};
    uint64_t strides[2] = {(uint64_t)D * 2, (uint64_t)row_stride * 2};
    uint32_t box[3] = {64, 1, 128};
    return encode_tmap(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(q), dims, strides,
                       box, CU_TENSOR_MAP_SWIZZLE_128B);
}

static kvs_status check_arena(const kvs_kv_arena *a, int32_t num_heads) {
    KVS_REQUIRE(a != nullptr, KVS_EPARAM, "null arena");
    KVS_REQUIRE(a->head_dim == 128, KVS_ESHAPE, "tcgen05 attention needs head_dim == 128 (got %d)",
                a->head_dim);
    KVS_REQUIRE(a->page_size == 64, KVS_ESHAPE, "tcgen05 attention needs page_size == 64");
    KVS_REQUIRE(num_heads % a->kv_heads == 0, KVS_ESHAPE, "num_heads %% kv_heads != 0");
    return KVS_OK;
}

template <bool kPV>
static size_t fwd_smem() {
    return 1024 + attn::TILE_BYTES * (1 + attn::NS + (kPV ? attn::NS + 2 : 0));
}

}  // namespace kvs

using namespace kvs;

static kvs_status attention_fwd_impl(const void *q, int64_t q_row_stride, const kvs_rope *rope,
                                     const int32_t *row_pos, int64_t n_rows, int32_t num_heads,
                                     const int32_t *tile_req, const int32_t *tile_row0,
                                     const int32_t *tile_rows, int32_t n_tiles,
                                     const int32_t *kv_len, int32_t causal, int32_t layer,
                                     const kvs_kv_arena *arena, const kvs_batch *batch,
                                     float softmax_scale, void *out, float *lse,
                                     kvs_stream_t stream) {
    kvs_status st = check_arena(arena, num_heads);
    if (st != KVS_OK) return st;
    KVS_REQUIRE(batch != nullptr, KVS_EPARAM, "null batch");
    KVS_REQUIRE(causal || kv_len != nullptr, KVS_EPARAM, "non-causal attention needs kv_len");
    KVS_REQUIRE(rope == nullptr || (rope->cos != nullptr && rope->sin != nullptr), KVS_EPARAM,
                "rope tables are null");
    KVS_REQUIRE(rope == nullptr || ((((uintptr_t)rope->cos) | ((uintptr_t)rope->sin)) & 15) == 0,
                KVS_EPARAM, "rope tables must be 16-byte aligned");
    KVS_REQUIRE(q_row_stride >= (int64_t)num_heads * 128 && q_row_stride % 8 == 0, KVS_ESHAPE,
                "q row stride %lld below H*128 or not 16-byte aligned", (long long)q_row_stride);
    if (n_tiles <= 0 || n_rows <= 0) return KVS_OK;
    KVS_REQUIRE(n_tiles <= 65535, KVS_ESHAPE, "more than 65535 row tiles in one launch");
    CUtensorMap mq, mkv;
    KVS_REQUIRE(make_q_map(&mq, q, n_rows, num_heads, 128, q_row_stride), KVS_ECUDA,
                "Q tensor map");
    KVS_REQUIRE(make_kv_map(&mkv, arena), KVS_ECUDA, "KV tensor map");
    attn::Params p;
    p.row_pos = row_pos;
    p.tile_req = tile_req;
    p.tile_row0 = tile_row0;
    p.tile_rows = tile_rows;
    p.kv_len = kv_len;
    p.block_table = batch->block_table;
    p.max_pages = batch->max_pages;
    p.page_size = arena->page_size;
    p.num_layers = arena->num_layers;
    p.layer = layer;
    p.num_heads = num_heads;
    p.kv_heads = arena->kv_heads;
    p.causal = causal;
    p.scale_log2 = softmax_scale * 1.4426950408889634f;
    p.out = (__nv_bfloat16 *)out;
    p.lse = lse;
    p.n_rows = n_rows;
    p.q_cos = rope != nullptr ? rope->cos : nullptr;
    p.q_sin = rope != nullptr ? rope->sin : nullptr;
    static std::atomic<int> sched_next{0};
    p.sched = sched_next.fetch_add(1, std::memory_order_relaxed) & (attn::kSchedSlots - 1);
    cudaStream_t s = (cudaStream_t)stream;
    const int group = num_heads / arena->kv_heads;
    const char *variant = getenv("KVS_ATTN");
    // default: persistent head pairs (fwdp) for even GQA groups, persistent
    // single heads with double-buffered S (fwd6p; fwd6 when Q is rotated in
    // the kernel) otherwise; KVS_ATTN=1|3|6|p|q pins a variant (1: the
    // single-head kernel with P through shared memory, 3 / 6: one-shot CTAs)
    p.ppg = group / 2;
    p.h_stride = 1;
    p.h_offset = 0;
    p.h_count = num_heads;
    // odd groups > 1 (Qwen: 7): head pairs for all but the last head of each group
    // (fwdp), then that head alone (fwd6p) - 'm'
    const char v = variant != nullptr ? variant[0]
                   : (group % 2 == 0 ? 'p' : (group > 1 && rope == nullptr ? 'm' : 'q'));
    if (out != nullptr && rope == nullptr && v == 'm' && group % 2 != 0 && group > 1) {
        p.ppg = (group - 1) / 2;
        const size_t smem_p = 1024 + attn::TILE_BYTES * (2 + attn::RING3);
        cudaFuncSetAttribute(attn::fwdp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem_p);
        const int n_pairs = n_tiles * arena->kv_heads * p.ppg;
        attn::fwdp_kernel<<<std::min(n_pairs, kNumSMs), attn::kThreads2, smem_p, s>>>(mq, mkv, p,
                                                                                    n_pairs);
        p.h_stride = group;
        p.h_offset = group - 1;
        p.h_count = arena->kv_heads;
        p.sched = (p.sched + 1) & (attn::kSchedSlots - 1);
        const size_t smem_q = 1024 + attn::TILE_BYTES * (2 + attn::RING6P);
        cudaFuncSetAttribute(attn::fwd6p_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem_q);
        const int n_single = n_tiles * arena->kv_heads;
        attn::fwd6p_kernel<<<std::min(n_single, kNumSMs), attn::kThreads6, smem_q, s>>>(
            mq, mkv, p, n_single);
    } else if (out != nullptr && rope == nullptr && (v == 'q' || ((v == 'p' || v == 'm') && group % 2 != 0))) {
        const size_t smem = 1024 + attn::TILE_BYTES * (2 + attn::RING6P);
        cudaFuncSetAttribute(attn::fwd6p_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        const int n_items = n_tiles * num_heads;
        attn::fwd6p_kernel<<<std::min(n_items, kNumSMs), attn::kThreads6, smem, s>>>(mq, mkv, p,
                                                                                    n_items);
    } else if (out != nullptr && (v == '6' || v == 'q' || (v != '1' && group % 2 != 0))) {
        const size_t smem = 1024 + attn::TILE_BYTES * (1 + attn::RING6);
        cudaFuncSetAttribute(attn::fwd6_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        attn::fwd6_kernel<<<dim3(num_heads, n_tiles), attn::kThreads6, smem, s>>>(mq, mkv, p);
    } else if (out != nullptr && group % 2 == 0 && v == 'p') {
        const size_t smem = 1024 + attn::TILE_BYTES * (2 + attn::RING3);
        cudaFuncSetAttribute(attn::fwdp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        const int n_items = n_tiles * (num_heads / 2);
        attn::fwdp_kernel<<<std::min(n_items, kNumSMs), attn::kThreads2, smem, s>>>(mq, mkv, p,
                                                                                  n_items);
    } else if (out != nullptr && group % 2 == 0 && v == '3') {
        const size_t smem = 1024 + attn::TILE_BYTES * (2 + attn::RING3);
        cudaFuncSetAttribute(attn::fwd3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        attn::fwd3_kernel<<<dim3(num_heads / 2, n_tiles), attn::kThreads2, smem, s>>>(mq, mkv, p);
    } else if (rope != nullptr) {
        KVS_REQUIRE(false, KVS_EPARAM, "in-kernel Q rotation needs the fwd3/fwd6 kernels");
    } else if (out != nullptr) {
        const size_t smem = fwd_smem<true>();
        cudaFuncSetAttribute(attn::fwd_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        attn::fwd_kernel<true><<<dim3(num_heads, n_tiles), attn::kThreads, smem, s>>>(mq, mkv, p);
    } else {
        const size_t smem = fwd_smem<false>();
        cudaFuncSetAttribute(attn::fwd_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        attn::fwd_kernel<false><<<dim3(num_heads, n_tiles), attn::kThreads, smem, s>>>(mq, mkv, p);
    }
    KVS_CHECK_LAUNCH("kvs_attention_fwd");
    return KVS_OK;
}

extern "C" {

kvs_status kvs_attention_fwd(const void *q, const int32_t *row_pos, int64_t n_rows,
                             int32_t num_heads, const int32_t *tile_req, const int32_t *tile_row0,
                             const int32_t *tile_rows, int32_t n_tiles, const int32_t *kv_len,
                             int32_t causal, int32_t layer, const kvs_kv_arena *arena,
                             const kvs_batch *batch, float softmax_scale, void *out, float *lse,
                             kvs_stream_t stream) {
    return attention_fwd_impl(q, (int64_t)num_heads * 128, nullptr, row_pos, n_rows, num_heads,
                              tile_req, tile_row0, tile_rows, n_tiles, kv_len, causal, layer,
                              arena, batch, softmax_scale, out, lse, stream);
}

kvs_status kvs_attention_fwd_qkv(const void *qkv, int64_t qkv_row_stride, const kvs_rope *rope,
                                 const int32_t *row_pos, int64_t n_rows, int32_t num_heads,
                                 const int32_t *tile_req, const int32_t *tile_row0,
                                 const int32_t *tile_rows, int32_t n_tiles,
                                 const int32_t *kv_len, int32_t causal, int32_t layer,
                                 const kvs_kv_arena *arena, const kvs_batch *batch,
                                 float softmax_scale, void *out, kvs_stream_t stream) {
    KVS_REQUIRE(out != nullptr, KVS_EPARAM, "null out");
    return attention_fwd_impl(qkv, qkv_row_stride, rope, row_pos, n_rows, num_heads, tile_req,
                              tile_row0, tile_rows, n_tiles, kv_len, causal, layer, arena, batch,
                              softmax_scale, out, nullptr, stream);
}

int32_t kvs_attn_trace_dump(int64_t *host, int32_t max_pairs) {
#ifdef KVS_ATTN_TRACE
    static long long buf[64 * 256];
    cudaMemcpyFromSymbol(buf, attn::g_trace, sizeof(buf));
    int n = 0;
    for (int i = 0; i < 64 * 256 && n < max_pairs; ++i)
        if (buf[i] != 0) {
            host[2 * n] = buf[i];
            host[2 * n + 1] = ((long long)(i / 256) << 32) | (i % 256);
            ++n;
        }
    static long long zero[64 * 256];
    cudaMemcpyToSymbol(attn::g_trace, zero, sizeof(zero));
    return n;
#else
    (void)host;
    (void)max_pairs;
    return -1;
#endif
}

size_t kvs_dhd_alpha_workspace(int64_t n_total, int32_t num_heads, int32_t kv_heads) {
    return ((sizeof(float) * (size_t)n_total * num_heads + 255) & ~(size_t)255) +
           sizeof(float) * (size_t)n_total * kv_heads;
}

kvs_status kvs_dhd_alpha(const void *q, int32_t num_heads, int32_t causal, int32_t layer,
                         const kvs_kv_arena *arena, const kvs_batch *batch,
                         const int32_t *row_pos, const int32_t *tile_req,
                         const int32_t *tile_row0, const int32_t *tile_rows, int32_t n_tiles,
                         const int32_t *kv_len, float softmax_scale, float *alpha, void *ws,
                         size_t ws_bytes, kvs_stream_t stream) {
    kvs_status st = check_arena(arena, num_heads);
    if (st != KVS_OK) return st;
    KVS_REQUIRE(batch != nullptr, KVS_EPARAM, "null batch");
    KVS_REQUIRE(causal || kv_len != nullptr, KVS_EPARAM, "non-causal alpha needs kv_len");
    const int64_t n_total = batch->n_total;
    KVS_REQUIRE(ws_bytes >= kvs_dhd_alpha_workspace(n_total, num_heads, arena->kv_heads),
                KVS_EPARAM, "workspace too small");
    if (n_tiles <= 0 || n_total <= 0) return KVS_OK;
    float *lse = (float *)ws;
    float *part = (float *)((char *)ws + (((sizeof(float) * (size_t)n_total * num_heads) + 255) &
                                          ~(size_t)255));
    cudaStream_t s = (cudaStream_t)stream;
    // pass 1: row log-sum-exp (the forward kernel without P.V)
    st = kvs_attention_fwd(q, row_pos, n_total, num_heads, tile_req, tile_row0, tile_rows, n_tiles,
                           kv_len, causal, layer, arena, batch, softmax_scale, nullptr, lse,
                           stream);
    if (st != KVS_OK) return st;
    // pass 2: key-major column sums
    CUtensorMap mq, mkv;
    KVS_REQUIRE(make_q_map(&mq, q, n_total, num_heads, 128), KVS_ECUDA, "Q tensor map");
    KVS_REQUIRE(make_kv_map(&mkv, arena), KVS_ECUDA, "KV tensor map");
    attn::ColParams cp;
    cp.req_off = batch->req_off;
    cp.row_pos = row_pos;
    cp.tile_req = tile_req;
    cp.tile_row0 = tile_row0;
    cp.lse = lse;
    cp.block_table = batch->block_table;
    cp.max_pages = batch->max_pages;
    cp.page_size = arena->page_size;
    cp.num_layers = arena->num_layers;
    cp.layer = layer;
    cp.num_heads = num_heads;
    cp.kv_heads = arena->kv_heads;
    cp.causal = causal;
    cp.scale_log2 = softmax_scale * 1.4426950408889634f;
    cp.alpha_part = part;
    const size_t smem = 1024 + attn::TILE_BYTES * (1 + attn::NS);
    cudaFuncSetAttribute(attn::colsum_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    attn::colsum_kernel<<<dim3(n_tiles, arena->kv_heads), attn::kThreads, smem, s>>>(mq, mkv, cp);
    attn::alpha_reduce_kernel<<<kNumSMs * 4, 256, 0, s>>>(part, n_total, arena->kv_heads,
                                                         num_heads, alpha);
    KVS_CHECK_LAUNCH("kvs_dhd_alpha");
    return KVS_OK;
}

}  // extern "C"
