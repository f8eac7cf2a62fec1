// Few-row attention for decode steps and probe queries (kvs_decode_attention):
// the per-token attention of _token_rows (reference engine.py:104-109) for
// rows that each attend to their own request's paged K/V up to their own
// position (causal) or kv_len.
//
// The bound is HBM: a decode step's rows are a request's new token plus the
// rows D3 chose for recompute, all reading the same context.  So a CTA owns
// a CHUNK of up to 16 / group consecutive rows (rows of one request are
// contiguous in every caller) and one kv head; the chunk's rows x the group's
// query heads are the 16 M rows of mma.sync m16n8k16 tiles, and every K/V
// page of the request is read once for all of them (the SIMT kernel this
// replaces read it once per row).  Runs of rows of different requests inside
// a chunk (probe queries: one row per request) are processed one after the
// other with the other runs' M rows masked.
//
// Per warp, flash-decoding over whole 64-key pages: K and V of one kv head
// arrive by TMA (SWIZZLE_128B, 16 KB each) into the warp's own 2-stage ring
// (no producer warp), S = Q.K^T (16 x 64) with ldmatrix + mma.sync, masked
// online softmax on the C fragments (quad shuffles), P re-packed in
// registers as the A operand of O += P.V (ldmatrix.trans on the V tile).
// Keys are split over (pages of the run) x splits x warps; the CTA's warps
// merge through shared memory into the same (m, l, O) split partials the
// combine kernel reduces.
#include "common.cuh"

namespace kvs {
namespace dattn {

constexpr int D = 128;
constexpr int kWarps = 3;
constexpr int kThreads = 32 * kWarps;
constexpr int kStages = 2;
constexpr int kPage = 64;                       // keys per page (arena page_size)
constexpr int kHalf = kPage * 128;              // one SW128 half tile: 64 rows x 64 dims bf16
constexpr int kTile = 2 * kHalf;                // 64 keys x 128 dims
constexpr int kStageBytes = 2 * kTile;          // K + V
constexpr int kMaxRuns = 16;

struct Smem {
    alignas(1024) uint8_t ring[kWarps][kStages][kStageBytes];
    alignas(1024) uint8_t q[16 * D * 2];          // 16 query vectors, SW128 (2 halves)
    uint64_t full[kWarps][kStages];
    int32_t run_req[kMaxRuns], run_row0[kMaxRuns], run_rows[kMaxRuns];
    int32_t run_page0[kMaxRuns], run_pages[kMaxRuns], run_kend[kMaxRuns];
    int32_t item_off[kMaxRuns + 1];
    int32_t row_kend[16];                       // per chunk row: keys [0, kend)
    int32_t n_runs;
};

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t &a0, uint32_t &a1, uint32_t &a2,
                                        uint32_t &a3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
                 : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3)
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t &a0, uint32_t &a1, uint32_t &a2,
                                          uint32_t &a3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
                 : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3)
                 : "r"(addr));
}
__device__ __forceinline__ void mma16816(float *c, uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 "
        "{%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, {%0, %1, %2, %3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
// byte offset of 16-byte chunk `chunk` (dims 8*chunk..+8) of row `row` in a
// [rows x 128 dims] tile stored as two SW128 halves of [rows x 64 dims]
__device__ __forceinline__ uint32_t sw_off(int row, int chunk, int rows) {
    return (uint32_t)((chunk >> 3) * rows * 128 + row * 128 + (((chunk & 7) ^ (row & 7)) << 4));
}

struct Params {
    const __nv_bfloat16 *q;
    const int32_t *row_req, *row_pos, *kv_len;
    int64_t n_rows;
    int32_t H, G, causal, layer, num_layers, page_size;
    const int32_t *block_table;
    int32_t max_pages, splits;
    float scale_log2;
    float *ws;                                  // [row][H][splits][D + 2]: m, l, O
};

template <int HQ>
__global__ void __launch_bounds__(kThreads, 1)
    decode_attn_tc_kernel(const __grid_constant__ CUtensorMap map_kv, const Params p) {
    constexpr int RT = 16 / HQ;                 // rows per chunk
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    Smem &sm = *reinterpret_cast<Smem *>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int chunk = blockIdx.x, g = blockIdx.y, split = blockIdx.z;
    const int64_t row0 = (int64_t)chunk * RT;
    const int nrows = (int)min((int64_t)RT, p.n_rows - row0);
    // ---- runs of rows of one request; each run's pages of this split
    if (tid == 0) {
        int n = 0;
        for (int i = 0; i < nrows; ++i) {
            const int r = p.row_req[row0 + i];
            const int ke = p.causal ? p.row_pos[row0 + i] + 1 : p.kv_len[r];
            sm.row_kend[i] = ke;
            if (n > 0 && sm.run_req[n - 1] == r) {
                ++sm.run_rows[n - 1];
                sm.run_kend[n - 1] = max(sm.run_kend[n - 1], ke);
            } else {
                sm.run_req[n] = r;
                sm.run_row0[n] = i;
                sm.run_rows[n] = 1;
                sm.run_kend[n] = ke;
                ++n;
            }
        }
        int acc = 0;
        for (int u = 0; u < n; ++u) {
            const int pages = (sm.run_kend[u] + kPage - 1) / kPage;
            const int per = (pages + p.splits - 1) / p.splits;
            const int a = min(pages, split * per), b = min(pages, a + per);
            sm.run_page0[u] = a;
            sm.run_pages[u] = b - a;
            sm.item_off[u] = acc;
            acc += b - a;
        }
        sm.item_off[n] = acc;
        sm.n_runs = n;
        for (int w = 0; w < kWarps; ++w)
            for (int s = 0; s < kStages; ++s) mbar_init(&sm.full[w][s], 1);
        fence_barrier_init();
    }
    // ---- the chunk's query vectors: M row m = (chunk row m / HQ, head m % HQ)
    for (int e = tid; e < 16 * 16; e += kThreads) {
        const int m = e >> 4, c = e & 15;
        uint4 v = make_uint4(0u, 0u, 0u, 0u);
        if (m < nrows * HQ)
            v = *reinterpret_cast<const uint4 *>(
                p.q + ((row0 + m / HQ) * p.H + g * HQ + m % HQ) * D + 8 * c);
        *reinterpret_cast<uint4 *>(sm.q + sw_off(m, c, 16)) = v;
    }
    __syncthreads();
    const int n_items = sm.item_off[sm.n_runs];
    // item k (run-major over the runs' pages) -> warp k % kWarps
    auto locate = [&](int k, int &u, int &pg) {
        u = 0;
        while (sm.item_off[u + 1] <= k) ++u;
        pg = sm.run_page0[u] + (k - sm.item_off[u]);
    };
    auto issue = [&](int j, int s) {
        const int k = warp + j * kWarps;
        if (lane != 0 || k >= n_items) return;
        int u, pg;
        locate(k, u, pg);
        const int page = __ldg(p.block_table + (int64_t)sm.run_req[u] * p.max_pages + pg);
        uint8_t *dst = sm.ring[warp][s];
        uint64_t *bar = &sm.full[warp][s];
        fence_proxy_async_smem();
        mbar_expect_tx(bar, kStageBytes);
        const int c3 = (page * p.num_layers + p.layer) * 2;
        for (int kv = 0; kv < 2; ++kv)
            for (int hf = 0; hf < 2; ++hf)
                tma_load_4d(dst + kv * kTile + hf * kHalf, &map_kv, bar, hf * 64, g, 0, c3 + kv);
    };
    for (int s = 0; s < kStages; ++s) issue(s, s);
    __syncwarp();
    // Q as the A operand of every S tile: 8 k-steps of 16 dims
    uint32_t qa[8][4];
    {
        const uint32_t qbase = smem_u32(sm.q);
        const int mi = lane >> 3;
        const int row = (mi & 1) * 8 + (lane & 7);
#pragma unroll
        for (int ks = 0; ks < 8; ++ks)
            ldsm_x4(qbase + sw_off(row, ks * 2 + (mi >> 1), 16), qa[ks][0], qa[ks][1], qa[ks][2],
                    qa[ks][3]);
    }
    // this thread's two M rows (C fragment rows lane/4 and lane/4 + 8)
    const int mr[2] = {lane >> 2, (lane >> 2) + 8};
    int mrow_chunk[2], mkend[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        mrow_chunk[h] = mr[h] < nrows * HQ ? mr[h] / HQ : -1;
        mkend[h] = mrow_chunk[h] >= 0 ? sm.row_kend[mrow_chunk[h]] : 0;
    }
    float m_run[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.f, 0.f};
    float o[16][4];
#pragma unroll
    for (int nb = 0; nb < 16; ++nb)
#pragma unroll
        for (int e = 0; e < 4; ++e) o[nb][e] = 0.f;
    for (int j = 0;; ++j) {
        const int k = warp + j * kWarps;
        if (k >= n_items) break;
        const int s = j % kStages;
        int u, pg;
        locate(k, u, pg);
        mbar_wait(&sm.full[warp][s], (uint32_t)(j / kStages) & 1u);
        const uint32_t kbase = smem_u32(sm.ring[warp][s]);
        const uint32_t vbase = kbase + kTile;
        // ---- S = Q . K^T over the page's 64 keys: 8 n-blocks of 8 keys
        float sc[8][4];
#pragma unroll
        for (int nb = 0; nb < 8; ++nb) {
#pragma unroll
            for (int e = 0; e < 4; ++e) sc[nb][e] = 0.f;
            const int mi = lane >> 3;
            const int key = nb * 8 + (lane & 7);
#pragma unroll
            for (int kp = 0; kp < 4; ++kp) {
                uint32_t b0, b1, b2, b3;                 // k-steps 2kp (b0, b1), 2kp+1 (b2, b3)
                ldsm_x4(kbase + sw_off(key, kp * 4 + mi, kPage), b0, b1, b2, b3);
                mma16816(sc[nb], qa[2 * kp][0], qa[2 * kp][1], qa[2 * kp][2], qa[2 * kp][3], b0, b1);
                mma16816(sc[nb], qa[2 * kp + 1][0], qa[2 * kp + 1][1], qa[2 * kp + 1][2],
                         qa[2 * kp + 1][3], b2, b3);
            }
        }
        __syncwarp();
        // ---- mask (run membership, causal end) and online softmax per M row
        const int key0 = (sm.run_page0[u] + (k - sm.item_off[u])) * kPage;
        const int r0 = sm.run_row0[u], r1 = r0 + sm.run_rows[u];
        float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const bool in_run = mrow_chunk[h] >= r0 && mrow_chunk[h] < r1;
#pragma unroll
            for (int nb = 0; nb < 8; ++nb)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int key = key0 + nb * 8 + 2 * (lane & 3) + e;
                    float &x = sc[nb][2 * h + e];
                    x = (in_run && key < mkend[h]) ? x * p.scale_log2 : -INFINITY;
                    mx[h] = fmaxf(mx[h], x);
                }
            mx[h] = fmaxf(mx[h], __shfl_xor_sync(0xffffffffu, mx[h], 1));
            mx[h] = fmaxf(mx[h], __shfl_xor_sync(0xffffffffu, mx[h], 2));
        }
        float corr[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const float mn = fmaxf(m_run[h], mx[h]);
            corr[h] = (mn == -INFINITY || m_run[h] == -INFINITY) ? (mn == -INFINITY ? 1.f : 0.f)
                                                                 : fast_exp2(m_run[h] - mn);
            const float mu = mn == -INFINITY ? 0.f : mn;
            float ls = 0.f;
#pragma unroll
            for (int nb = 0; nb < 8; ++nb)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    float &x = sc[nb][2 * h + e];
                    x = fast_exp2(x - mu);                  // -inf -> 0
                    ls += x;
                }
            ls += __shfl_xor_sync(0xffffffffu, ls, 1);
            ls += __shfl_xor_sync(0xffffffffu, ls, 2);
            l_run[h] = l_run[h] * corr[h] + ls;
            m_run[h] = mn;
        }
#pragma unroll
        for (int nb = 0; nb < 16; ++nb) {
            o[nb][0] *= corr[0];
            o[nb][1] *= corr[0];
            o[nb][2] *= corr[1];
            o[nb][3] *= corr[1];
        }
        // ---- O += P . V: 4 k-steps of 16 keys, 16 n-blocks of 8 dims
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
            const uint32_t a0 = pack_bf16x2(sc[2 * kk][0], sc[2 * kk][1]);
            const uint32_t a1 = pack_bf16x2(sc[2 * kk][2], sc[2 * kk][3]);
            const uint32_t a2 = pack_bf16x2(sc[2 * kk + 1][0], sc[2 * kk + 1][1]);
            const uint32_t a3 = pack_bf16x2(sc[2 * kk + 1][2], sc[2 * kk + 1][3]);
            const int mi = lane >> 3;
            const int key = kk * 16 + (mi & 1) * 8 + (lane & 7);
#pragma unroll
            for (int np = 0; np < 8; ++np) {             // n-blocks 2np (b0, b1), 2np+1 (b2, b3)
                uint32_t b0, b1, b2, b3;
                ldsm_x4_t(vbase + sw_off(key, np * 2 + (mi >> 1), kPage), b0, b1, b2, b3);
                mma16816(o[2 * np], a0, a1, a2, a3, b0, b1);
                mma16816(o[2 * np + 1], a0, a1, a2, a3, b2, b3);
            }
        }
        __syncwarp();
        issue(j + kStages, s);                           // the stage is free again
    }
    // ---- merge the warps' (m, l, O) per M row through shared memory (ring reused)
    __syncthreads();
    float *so = reinterpret_cast<float *>(&sm.ring[0][0][0]);          // [warp][16][D]
    float *sml = so + kWarps * 16 * D;                                   // [warp][16][2]
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        if ((lane & 3) == 0) {
            sml[(warp * 16 + mr[h]) * 2 + 0] = m_run[h];
            sml[(warp * 16 + mr[h]) * 2 + 1] = l_run[h];
        }
#pragma unroll
        for (int nb = 0; nb < 16; ++nb) {
            const int col = nb * 8 + 2 * (lane & 3);
            so[(warp * 16 + mr[h]) * D + col] = o[nb][2 * h];
            so[(warp * 16 + mr[h]) * D + col + 1] = o[nb][2 * h + 1];
        }
    }
    __syncthreads();
    for (int e = tid; e < nrows * HQ * D; e += kThreads) {
        const int m = e / D, d = e - m * D;
        float M = -INFINITY;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) M = fmaxf(M, sml[(w * 16 + m) * 2]);
        float L = 0.f, S = 0.f;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            const float mw = sml[(w * 16 + m) * 2];
            if (mw == -INFINITY) continue;
            const float c = fast_exp2(mw - M);
            L += sml[(w * 16 + m) * 2 + 1] * c;
            S += so[(w * 16 + m) * D + d] * c;
        }
        const int64_t row = row0 + m / HQ;
        float *out = p.ws + ((row * p.H + g * HQ + m % HQ) * p.splits + split) * (D + 2);
        if (d == 0) {
            out[0] = M;
            out[1] = L;
        }
        out[2 + d] = S;
    }
}

__global__ void combine_kernel(const float *__restrict__ ws, int32_t H, int32_t n_splits,
                               __nv_bfloat16 *__restrict__ out) {
    const int64_t row = blockIdx.x;
    const int h = blockIdx.y, d = threadIdx.x;
    const float *base = ws + (row * H + h) * n_splits * (D + 2);
    float M = -INFINITY;
    for (int sp = 0; sp < n_splits; ++sp) M = fmaxf(M, base[sp * (D + 2)]);
    float L = 0.f, S = 0.f;
    for (int sp = 0; sp < n_splits; ++sp) {
        const float *o = base + sp * (D + 2);
        if (o[0] == -INFINITY) continue;
        const float c = fast_exp2(o[0] - M);
        L += o[1] * c;
        S += o[2 + d] * c;
    }
    out[(row * H + h) * D + d] = f2bf(L > 0.f ? S / L : 0.f);
}

// splits: every CTA pays a fixed prologue (runs, Q tile, barriers, first
// TMA round trip) and epilogue (warp merge), so a launch should be ONE wave
// of CTAs when the (chunk, kv head) pairs allow it, each split as long as
// possible; larger batches take the split count with the best wave fill.
static int splits_for(int64_t n_rows, int H, int G, int max_kv) {
    const int hq = H / G, rt = 16 / hq;
    const int64_t pairs = ((n_rows + rt - 1) / rt) * G;
    const int cap = (max_kv + 2 * kPage - 1) / (2 * kPage);             // >= 2 pages per split
    if (pairs >= kNumSMs) return 1;
    int64_t s = kNumSMs / pairs;
    if (s > cap) s = cap;
    if (s > 64) s = 64;
    return s < 1 ? 1 : (int)s;
}

}  // namespace dattn

}  // namespace kvs

using namespace kvs;

extern "C" {

size_t kvs_decode_attention_workspace(int64_t n_rows, int32_t num_heads, int32_t kv_heads,
                                      int32_t head_dim, int32_t max_kv) {
    if (kv_heads <= 0 || num_heads % kv_heads != 0) return 0;
    const int splits = dattn::splits_for(n_rows, num_heads, kv_heads, max_kv);
    return sizeof(float) * (size_t)n_rows * num_heads * splits * (head_dim + 2);
}

kvs_status kvs_decode_attention(const void *q, const int32_t *row_req, const int32_t *row_pos,
                                int64_t n_rows, int32_t num_heads, const int32_t *kv_len,
                                int32_t causal, int32_t layer, const kvs_kv_arena *arena,
                                const kvs_batch *batch, float softmax_scale, void *out, void *ws,
                                size_t ws_bytes, kvs_stream_t stream) {
    KVS_REQUIRE(arena && batch, KVS_EPARAM, "null arena/batch");
    const int G = arena->kv_heads, Dh = arena->head_dim;
    KVS_REQUIRE(num_heads % G == 0 && num_heads / G <= 8, KVS_ESHAPE,
                "num_heads / kv_heads must be <= 8");
    KVS_REQUIRE(Dh == 128, KVS_ESHAPE, "decode attention needs head_dim == 128 (padded heads)");
    KVS_REQUIRE(arena->page_size == dattn::kPage, KVS_ESHAPE, "decode attention needs page_size 64");
    KVS_REQUIRE(causal || kv_len != nullptr, KVS_EPARAM, "non-causal attention needs kv_len");
    if (n_rows <= 0) return KVS_OK;
    const int max_kv = batch->max_pages * arena->page_size;
    const int splits = dattn::splits_for(n_rows, num_heads, G, max_kv);
    KVS_REQUIRE(ws_bytes >= sizeof(float) * (size_t)n_rows * num_heads * splits * (Dh + 2),
                KVS_EPARAM, "workspace too small");
    CUtensorMap mkv;
    KVS_REQUIRE(make_kv_map(&mkv, arena), KVS_ECUDA, "KV tensor map");
    dattn::Params p;
    p.q = (const __nv_bfloat16 *)q;
    p.row_req = row_req;
    p.row_pos = row_pos;
    p.kv_len = kv_len;
    p.n_rows = n_rows;
    p.H = num_heads;
    p.G = G;
    p.causal = causal;
    p.layer = layer;
    p.num_layers = arena->num_layers;
    p.page_size = arena->page_size;
    p.block_table = batch->block_table;
    p.max_pages = batch->max_pages;
    p.splits = splits;
    p.scale_log2 = softmax_scale * 1.4426950408889634f;
    p.ws = (float *)ws;
    cudaStream_t s = (cudaStream_t)stream;
    const int hq = num_heads / G;
    const size_t smem = sizeof(dattn::Smem) + 1024;
    const unsigned chunks = (unsigned)((n_rows + (16 / hq) - 1) / (16 / hq));
    const dim3 grid(chunks, G, splits);
#define KVS_DATTN(HQ)                                                                         \
    cudaFuncSetAttribute(dattn::decode_attn_tc_kernel<HQ>,                                    \
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);             \
    dattn::decode_attn_tc_kernel<HQ><<<grid, dattn::kThreads, smem, s>>>(mkv, p)
    switch (hq) {
        case 1: KVS_DATTN(1); break;
        case 2: KVS_DATTN(2); break;
        case 3: KVS_DATTN(3); break;
        case 4: KVS_DATTN(4); break;
        case 5: KVS_DATTN(5); break;
        case 6: KVS_DATTN(6); break;
        case 7: KVS_DATTN(7); break;
        default: KVS_DATTN(8); break;
    }
#undef KVS_DATTN
    dattn::combine_kernel<<<dim3((unsigned)n_rows, num_heads), Dh, 0, s>>>(
        (const float *)ws, num_heads, splits, (__nv_bfloat16 *)out);
    KVS_CHECK_LAUNCH("kvs_decode_attention");
    return KVS_OK;
}

}  // extern "C"
