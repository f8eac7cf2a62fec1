// G1 reused-KV gather with fused RoPE re-alignment, the post-GEMM q/k/v
// RoPE + paged scatter, embedding rows and the recompute row-set builder.
//
// Reference: cached-row substitution model.py:196-200 / engine.py:204-206
// (K and V rows of every layer copied verbatim from the entry); RoPE is an
// extension: K is kept post-rotation at the owner's positions
// and re-aligned by the rotation of (dst_pos - cand_pos).
#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace kvs {

struct Arena {
    __nv_bfloat16 *base;
    int32_t L, G, D, P;  // layers, kv heads, head dim, page size
    __device__ __forceinline__ __nv_bfloat16 *row(int64_t page, int layer, int kv, int r) const {
        return base + ((((size_t)page * L + layer) * 2 + kv) * P + r) * (size_t)(G * D);
    }
};

static inline Arena make_arena(const kvs_kv_arena *a) {
    return Arena{(__nv_bfloat16 *)a->base, a->num_layers, a->kv_heads, a->head_dim, a->page_size};
}

// Rotate-half RoPE on 8 consecutive dims [8c, 8c+8) of the first half paired
// with [half + 8c, ...): angle index delta (cos even, sin odd).
__device__ __forceinline__ void rope8(const uint4 &lo_in, const uint4 &hi_in, uint4 &lo_out,
                                      uint4 &hi_out, const float *__restrict__ cos_t,
                                      const float *__restrict__ sin_t, int32_t delta, int half,
                                      int c) {
    const int32_t a = delta < 0 ? -delta : delta;
    const float sgn = delta < 0 ? -1.f : 1.f;
    const __nv_bfloat16 *x1 = reinterpret_cast<const __nv_bfloat16 *>(&lo_in);
    const __nv_bfloat16 *x2 = reinterpret_cast<const __nv_bfloat16 *>(&hi_in);
    const float4 c0 = *reinterpret_cast<const float4 *>(cos_t + (size_t)a * half + 8 * c);
    const float4 c1 = *reinterpret_cast<const float4 *>(cos_t + (size_t)a * half + 8 * c + 4);
    const float4 s0 = *reinterpret_cast<const float4 *>(sin_t + (size_t)a * half + 8 * c);
    const float4 s1 = *reinterpret_cast<const float4 *>(sin_t + (size_t)a * half + 8 * c + 4);
    const float cs[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
    const float sn[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
    uint32_t *o1 = reinterpret_cast<uint32_t *>(&lo_out);
    uint32_t *o2 = reinterpret_cast<uint32_t *>(&hi_out);
#pragma unroll
    for (int k = 0; k < 8; k += 2) {
        float a0 = bf2f(x1[k]), a1 = bf2f(x1[k + 1]);
        float b0 = bf2f(x2[k]), b1 = bf2f(x2[k + 1]);
        float s0v = sgn * sn[k], s1v = sgn * sn[k + 1];
        o1[k / 2] = pack_bf16x2(a0 * cs[k] - b0 * s0v, a1 * cs[k + 1] - b1 * s1v);
        o2[k / 2] = pack_bf16x2(b0 * cs[k] + a0 * s0v, b1 * cs[k + 1] + a1 * s1v);
    }
}

// One CTA per flat position; misses exit.  Each layer moves one K and one V
// row (G*D bf16) with 16-byte vector loads/stores; K rotated in registers.
// With slot_owner / peer_base (multi-GPU, peer memory): a slot owned by GPU r
// (slot_owner[slot] = r >= 0) is read straight from r's arena, mapped into
// this process (CUDA IPC; NVLink loads across GPUs), with the same page
// geometry - the remote fetch and the gather are one pass, no pack/exchange.
__global__ void __launch_bounds__(128) gather_kv_kernel(
    Arena A, const int64_t *__restrict__ req_off, int32_t n_req,
    const int32_t *__restrict__ block_table, int32_t max_pages,
    const int32_t *__restrict__ src_slot, const int32_t *__restrict__ src_cand,
    const int32_t *__restrict__ slot_pages, int32_t slot_max_pages, int32_t l0, int32_t l1,
    const float *__restrict__ cos_t, const float *__restrict__ sin_t,
    const int32_t *__restrict__ slot_owner, const unsigned long long *__restrict__ peer_base) {
    const int64_t t = blockIdx.x;
    const int32_t slot = src_slot[t];
    if (slot < 0) return;
    Arena S = A;                                  // where the source rows live
    if (slot_owner != nullptr) {
        const int32_t owner = slot_owner[slot];
        if (owner >= 0) S.base = reinterpret_cast<__nv_bfloat16 *>(peer_base[owner]);
    }
    int lo = 0, hi = n_req;
    while (hi - lo > 1) {
        int mid = (lo + hi) >> 1;
        if (req_off[mid] <= t) lo = mid; else hi = mid;
    }
    const int32_t pos = (int32_t)(t - req_off[lo]);
    const int32_t cand = src_cand[t];
    const int64_t dpage = block_table[(int64_t)lo * max_pages + pos / A.P];
    const int64_t spage = slot_pages[(int64_t)slot * slot_max_pages + cand / A.P];
    const int drow = pos % A.P, srow = cand % A.P;
    const int half = A.D / 2, chunks = half / 8;            // 16-byte chunks per half head
    const int kvec = A.G * chunks;                          // rotation work items per K row
    const int vvec = A.G * A.D / 8;                         // 16-byte vectors per V row
    const int32_t delta = pos - cand;
    for (int layer = l0; layer < l1; ++layer) {
        const uint4 *sk = reinterpret_cast<const uint4 *>(S.row(spage, layer, 0, srow));
        const uint4 *sv = reinterpret_cast<const uint4 *>(S.row(spage, layer, 1, srow));
        uint4 *dk = reinterpret_cast<uint4 *>(A.row(dpage, layer, 0, drow));
        uint4 *dv = reinterpret_cast<uint4 *>(A.row(dpage, layer, 1, drow));
        for (int v = threadIdx.x; v < vvec; v += blockDim.x) dv[v] = sv[v];
        if (cos_t == nullptr || delta == 0) {
            for (int v = threadIdx.x; v < vvec; v += blockDim.x) dk[v] = sk[v];
        } else {
            for (int it = threadIdx.x; it < kvec; it += blockDim.x) {
                const int g = it / chunks, c = it % chunks;
                const int vlo = g * (A.D / 8) + c, vhi = vlo + chunks;
                uint4 lo_o, hi_o;
                rope8(sk[vlo], sk[vhi], lo_o, hi_o, cos_t, sin_t, delta, half, c);
                dk[vlo] = lo_o;
                dk[vhi] = hi_o;
            }
        }
    }
}

// One CTA per query row.  qkv row = [q (H*D) | k (G*D) | v (G*D)].  Work
// items: (H+G)*D/16 rotation items (two 16-byte vectors each) followed by
// G*D/8 V vectors; a thread takes two items per round and issues all of its
// loads (qkv vectors, then the row's cos/sin, which depend only on the
// position) before any arithmetic, so a CTA waits on two memory latencies.
__global__ void __launch_bounds__(256) qkv_rope_scatter_kernel(
    const __nv_bfloat16 *__restrict__ qkv, int32_t H, Arena A, const int32_t *__restrict__ row_req,
    const int32_t *__restrict__ row_pos, const uint8_t *__restrict__ write_kv, int32_t layer,
    const int32_t *__restrict__ block_table, int32_t max_pages, const float *__restrict__ cos_t,
    const float *__restrict__ sin_t, __nv_bfloat16 *__restrict__ q_out,
    __nv_bfloat16 *__restrict__ k_out, __nv_bfloat16 *__restrict__ v_out) {
    const int64_t row = blockIdx.x;
    const int G = A.G, D = A.D, half = D / 2, chunks = half / 8, vph = D / 8;
    const int64_t width = (int64_t)(H + 2 * G) * D;
    const uint4 *src = reinterpret_cast<const uint4 *>(qkv + row * width);
    const int32_t pos = __ldg(row_pos + row);
    const bool rope = cos_t != nullptr;
    const bool wkv = write_kv == nullptr || write_kv[row] != 0;
    uint4 *dk = nullptr, *dv = nullptr;
    if (wkv) {
        const int32_t r = row_req[row];
        const int64_t page = __ldg(block_table + (int64_t)r * max_pages + pos / A.P);
        dk = reinterpret_cast<uint4 *>(A.row(page, layer, 0, pos % A.P));
        dv = reinterpret_cast<uint4 *>(A.row(page, layer, 1, pos % A.P));
    }
    uint4 *qo = q_out ? reinterpret_cast<uint4 *>(q_out + row * (int64_t)H * D) : nullptr;
    uint4 *ko = k_out ? reinterpret_cast<uint4 *>(k_out + row * (int64_t)G * D) : nullptr;
    uint4 *vo = v_out ? reinterpret_cast<uint4 *>(v_out + row * (int64_t)G * D) : nullptr;
    const float4 *c4 = reinterpret_cast<const float4 *>(cos_t + (size_t)pos * half);
    const float4 *s4 = reinterpret_cast<const float4 *>(sin_t + (size_t)pos * half);
    // q_out == nullptr: the query heads are left to the attention kernel
    const int item0 = q_out != nullptr ? 0 : H * chunks;
    const int n_rope = (H + G) * chunks, n_items = n_rope + G * vph, vbase = (H + G) * vph;
    for (int base = item0; base < n_items; base += 2 * blockDim.x) {
        uint4 lo[2], hi[2];
        int it[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            it[u] = base + u * blockDim.x + threadIdx.x;
            if (it[u] < n_rope) {
                const int h = it[u] / chunks, c = it[u] % chunks;
                lo[u] = __ldcs(src + h * vph + c);
                hi[u] = __ldcs(src + h * vph + c + chunks);
            } else if (it[u] < n_items) {
                lo[u] = __ldcs(src + vbase + (it[u] - n_rope));
            }
        }
        float4 cs[2][2], sn[2][2];
#pragma unroll
        for (int u = 0; u < 2; ++u)
            if (rope && it[u] < n_rope) {
                const int c = it[u] % chunks;
                cs[u][0] = __ldg(c4 + 2 * c);
                cs[u][1] = __ldg(c4 + 2 * c + 1);
                sn[u][0] = __ldg(s4 + 2 * c);
                sn[u][1] = __ldg(s4 + 2 * c + 1);
            }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            if (it[u] < n_rope) {
                const int h = it[u] / chunks, c = it[u] % chunks;
                const int vlo = h * vph + c, vhi = vlo + chunks;
                uint4 a = lo[u], b = hi[u];
                if (rope) rope8_reg(lo[u], hi[u], a, b, cs[u][0], cs[u][1], sn[u][0], sn[u][1]);
                if (h < H) {
                    qo[vlo] = a;
                    qo[vhi] = b;
                } else {
                    const int kl = vlo - H * vph, kh = vhi - H * vph;
                    if (dk) { dk[kl] = a; dk[kh] = b; }
                    if (ko) { ko[kl] = a; ko[kh] = b; }
                }
            } else if (it[u] < n_items) {
                const int v = it[u] - n_rope;
                if (dv) dv[v] = lo[u];
                if (vo) vo[v] = lo[u];
            }
        }
    }
}

// Scatter v2 (the one launched): persistent CTAs, each walking rows
// blockIdx.x + k * gridDim.x.  A row's whole [q | k | v] slice (12 KB at
// Llama width) arrives with one TMA bulk copy into a kScatSlots-deep shared
// ring (2 slots x 128 threads: many small CTAs per SM beat deeper rings,
// 81 vs 104 us per session layer at 19.7k rows); warp 1 fetches the row's metadata (position, K/V destination) and
// its cos/sin coefficients into the slot kScatSlots-1 rows ahead, so the
// 256 consumer threads only read shared memory, rotate, and store.
#ifndef KVS_SCAT_SLOTS
#define KVS_SCAT_SLOTS 2
#endif
constexpr int kScatSlots = KVS_SCAT_SLOTS;
// a row's metadata is staged one iteration ahead and published by that
// iteration's closing barrier, so the ring needs at least two slots
static_assert(kScatSlots >= 2, "qkv_scatter2 needs at least two ring slots");
#ifndef KVS_SCAT_THREADS
#define KVS_SCAT_THREADS 128
#endif
constexpr int kScatThreads = KVS_SCAT_THREADS;

struct ScatMeta {
    int64_t dst;      // element offset of the row's K in the arena, -1: no K/V write
    int32_t pos;
    int32_t pad;
};

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes,
                                         uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__global__ void __launch_bounds__(kScatThreads) qkv_scatter2_kernel(
    const __nv_bfloat16 *__restrict__ qkv, int64_t n_rows, int32_t H, Arena A,
    const int32_t *__restrict__ row_req, const int32_t *__restrict__ row_pos,
    const uint8_t *__restrict__ write_kv, int32_t layer, const int32_t *__restrict__ block_table,
    int32_t max_pages, const float *__restrict__ cos_t, const float *__restrict__ sin_t,
    __nv_bfloat16 *__restrict__ q_out, __nv_bfloat16 *__restrict__ k_out,
    __nv_bfloat16 *__restrict__ v_out, const int32_t *__restrict__ src_row) {
    extern __shared__ __align__(128) uint8_t s_rows[];          // kScatSlots x row bytes
    __shared__ __align__(16) float s_cs[kScatSlots][2][64];
    __shared__ ScatMeta s_meta[kScatSlots];
    __shared__ __align__(8) uint64_t bars[kScatSlots];
    const int G = A.G, D = A.D, chunks = D / 16, vph = D / 8;
    const int64_t width = (int64_t)(H + 2 * G) * D;
    // q_out == nullptr: the query heads are left to the attention kernel and
    // only the row's k|v part is staged (4 of 12 KB at Llama width)
    const int64_t col0 = q_out != nullptr ? 0 : (int64_t)H * D;
    const uint32_t row_bytes = (uint32_t)((width - col0) * 2);
    const int tid = threadIdx.x;
    const int64_t n_mine = n_rows > (int64_t)blockIdx.x
                               ? (n_rows - 1 - (int64_t)blockIdx.x) / gridDim.x + 1 : 0;
    const bool rope = cos_t != nullptr;
    if (tid == 0) {
        for (int j = 0; j < kScatSlots; ++j) mbar_init(&bars[j], 1);
        fence_barrier_init();
    }
    __syncthreads();
    auto stage = [&](int64_t k) {                 // row k of this CTA into slot k % kScatSlots
        if (k >= n_mine) return;
        const int slot = (int)(k % kScatSlots);
        const int64_t row = (int64_t)blockIdx.x + k * gridDim.x;
        if (tid == 0) {
            mbar_expect_tx(&bars[slot], row_bytes);
            const int64_t src = src_row != nullptr ? (int64_t)src_row[row] : row;
            bulk_g2s(smem_u32(s_rows) + (uint32_t)slot * row_bytes, qkv + src * width + col0,
                     row_bytes, &bars[slot]);
        } else if (tid >= 32 && tid < 64) {
            const int lane = tid - 32;
            const int32_t pos = row_pos[row];
            if (lane == 0) {
                int64_t dst = -1;
                if (write_kv == nullptr || write_kv[row] != 0) {
                    const int64_t page = block_table[(int64_t)row_req[row] * max_pages + pos / A.P];
                    dst = A.row(page, layer, 0, pos % A.P) - A.base;
                }
                s_meta[slot] = ScatMeta{dst, pos, 0};
            }
            if (rope) {
                const float2 c = __ldg(reinterpret_cast<const float2 *>(cos_t + (size_t)pos * 64) + lane);
                const float2 sn = __ldg(reinterpret_cast<const float2 *>(sin_t + (size_t)pos * 64) + lane);
                reinterpret_cast<float2 *>(s_cs[slot][0])[lane] = c;
                reinterpret_cast<float2 *>(s_cs[slot][1])[lane] = sn;
            }
        }
    };
    for (int j = 0; j < kScatSlots - 1; ++j) stage(j);
    __syncthreads();
    const int item0 = q_out != nullptr ? 0 : H * chunks;
    const int n_rope = (H + G) * chunks, n_items = n_rope + G * vph, vbase = (H + G) * vph;
    for (int64_t k = 0; k < n_mine; ++k) {
        const int slot = (int)(k % kScatSlots);
        stage(k + kScatSlots - 1);                 // refills the slot freed last iteration
        mbar_wait(&bars[slot], (uint32_t)((k / kScatSlots) & 1));
        const int64_t row = (int64_t)blockIdx.x + k * gridDim.x;
        // staged vector v of the row is row vector v + col0 / 8
        const uint4 *src = reinterpret_cast<const uint4 *>(s_rows + (size_t)slot * row_bytes) -
                           col0 / 8;
        const ScatMeta m = s_meta[slot];
        uint4 *dk = m.dst >= 0 ? reinterpret_cast<uint4 *>(A.base + m.dst) : nullptr;
        uint4 *dv = m.dst >= 0 ? reinterpret_cast<uint4 *>(A.base + m.dst + (int64_t)A.P * G * D)
                               : nullptr;
        uint4 *qo = q_out ? reinterpret_cast<uint4 *>(q_out + row * (int64_t)H * D) : nullptr;
        uint4 *ko = k_out ? reinterpret_cast<uint4 *>(k_out + row * (int64_t)G * D) : nullptr;
        uint4 *vo = v_out ? reinterpret_cast<uint4 *>(v_out + row * (int64_t)G * D) : nullptr;
        const float *cs = s_cs[slot][0], *sn = s_cs[slot][1];
        for (int it = item0 + tid; it < n_items; it += blockDim.x) {
            if (it < n_rope) {
                const int h = it / chunks, c = it % chunks;
                const int vlo = h * vph + c, vhi = vlo + chunks;
                uint4 a = src[vlo], b = src[vhi];
                if (rope) {
                    const float4 c0 = *reinterpret_cast<const float4 *>(cs + 8 * c);
                    const float4 c1 = *reinterpret_cast<const float4 *>(cs + 8 * c + 4);
                    const float4 s0 = *reinterpret_cast<const float4 *>(sn + 8 * c);
                    const float4 s1 = *reinterpret_cast<const float4 *>(sn + 8 * c + 4);
                    uint4 lo_o, hi_o;
                    rope8_reg(a, b, lo_o, hi_o, c0, c1, s0, s1);
                    a = lo_o;
                    b = hi_o;
                }
                if (h < H) {
                    qo[vlo] = a;
                    qo[vhi] = b;
                } else {
                    const int kl = vlo - H * vph, kh = vhi - H * vph;
                    if (dk) { dk[kl] = a; dk[kh] = b; }
                    if (ko) { ko[kl] = a; ko[kh] = b; }
                }
            } else {
                const int v = it - n_rope;
                const uint4 x = src[vbase + v];
                if (dv) dv[v] = x;
                if (vo) vo[v] = x;
            }
        }
        __syncthreads();                           // slot consumed: the next stage() may refill it
    }
}

// out[r] = table[ids[r]] (rows of `width` bf16); out_f32 (optional) gets the
// same row widened to fp32 - the residual stream and the first layer's GEMM
// operand come out of one pass over the table rows.
__global__ void embed_rows_kernel(const __nv_bfloat16 *__restrict__ table, int64_t width,
                                  const int64_t *__restrict__ ids, const int32_t *__restrict__ rows,
                                  __nv_bfloat16 *__restrict__ out, float *__restrict__ out_f32) {
    const int64_t r = blockIdx.x;
    const int64_t id = ids[rows ? rows[r] : r];
    const uint4 *s = reinterpret_cast<const uint4 *>(table + id * width);
    uint4 *d = reinterpret_cast<uint4 *>(out + r * width);
    float4 *f = reinterpret_cast<float4 *>(out_f32 + r * width);
    for (int64_t v = threadIdx.x; v < width / 8; v += blockDim.x) {
        const uint4 x = __ldg(s + v);
        d[v] = x;
        if (out_f32 != nullptr) {
            const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&x);
            const float2 a = __bfloat1622float2(h[0]), b = __bfloat1622float2(h[1]);
            const float2 c = __bfloat1622float2(h[2]), e = __bfloat1622float2(h[3]);
            __stcs(f + 2 * v, make_float4(a.x, a.y, b.x, b.y));
            __stcs(f + 2 * v + 1, make_float4(c.x, c.y, e.x, e.y));
        }
    }
}

// Row set S = non-reused U selected U {n-1} of each request.
// Pass 1 (rows == nullptr): count per request.  Pass 2: compact in position
// order starting at row_off[r], emitting flat token index, request, position
// and whether the row's K/V are written fresh (non-reused or selected).
__global__ void __launch_bounds__(1024) build_rows_kernel(
    const int64_t *__restrict__ req_off, const int32_t *__restrict__ src_slot,
    const uint8_t *__restrict__ selected, int32_t *__restrict__ counts,
    const int64_t *__restrict__ row_off, int32_t *__restrict__ row_tok,
    int32_t *__restrict__ row_req, int32_t *__restrict__ row_pos, uint8_t *__restrict__ write_kv) {
    __shared__ int32_t warp_tot[32];
    __shared__ int32_t carry;
    const int r = blockIdx.x;
    const int64_t s = req_off[r], n = req_off[r + 1] - s;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int64_t base = 0; base < n; base += blockDim.x) {
        const int64_t i = base + threadIdx.x;
        bool in = false, fresh = false;
        if (i < n) {
            const bool reused = src_slot[s + i] >= 0;
            const bool sel = selected != nullptr && selected[s + i] != 0;
            fresh = !reused || sel;
            in = fresh || i == n - 1;
        }
        const uint32_t bal = __ballot_sync(0xffffffffu, in);
        const int before = __popc(bal & ((1u << lane) - 1));
        if (lane == 0) warp_tot[wid] = __popc(bal);
        __syncthreads();
        int wbase = 0, tot = 0;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
            if (k < wid) wbase += warp_tot[k];
            tot += warp_tot[k];
        }
        if (in && row_tok != nullptr) {
            const int64_t o = row_off[r] + carry + wbase + before;
            row_tok[o] = (int32_t)(s + i);
            row_req[o] = r;
            row_pos[o] = (int32_t)i;
            write_kv[o] = fresh ? 1 : 0;
        }
        __syncthreads();
        if (threadIdx.x == 0) carry += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0 && counts != nullptr) counts[r] = carry;
}

// X1 pack: rows (slot, cand) of the local pool -> dense [row][layer][K/V][G*D]
// for a peer that hit them (one CTA per row).
__global__ void __launch_bounds__(128) pack_rows_kernel(
    Arena A, const int32_t *__restrict__ slot, const int32_t *__restrict__ cand,
    const int32_t *__restrict__ slot_pages, int32_t slot_max_pages, uint4 *__restrict__ out) {
    const int64_t r = blockIdx.x;
    const int32_t s = slot[r], c = cand[r];
    const int64_t page = slot_pages[(int64_t)s * slot_max_pages + c / A.P];
    const int vvec = A.G * A.D / 8;
    uint4 *dst = out + r * (int64_t)A.L * 2 * vvec;
    for (int layer = 0; layer < A.L; ++layer)
        for (int kv = 0; kv < 2; ++kv) {
            const uint4 *src = reinterpret_cast<const uint4 *>(A.row(page, layer, kv, c % A.P));
            uint4 *d = dst + (layer * 2 + kv) * vvec;
            for (int v = threadIdx.x; v < vvec; v += blockDim.x) d[v] = src[v];
        }
}

// X1 unpack: dense rows received from peers -> the request's pages at flat
// position t[r], K re-aligned by (pos - cand[r]) (G1 semantics).
__global__ void __launch_bounds__(128) unpack_rows_kernel(
    Arena A, const int64_t *__restrict__ req_off, int32_t n_req,
    const int32_t *__restrict__ block_table, int32_t max_pages, const int64_t *__restrict__ flat_t,
    const int32_t *__restrict__ cand, const uint4 *__restrict__ in,
    const float *__restrict__ cos_t, const float *__restrict__ sin_t, int32_t layer_begin,
    int32_t layer_end, const uint8_t *__restrict__ skip) {
    const int64_t r = blockIdx.x;
    const int64_t t = flat_t[r];
    if (skip != nullptr && skip[t]) return;
    int lo = 0, hi = n_req;
    while (hi - lo > 1) {
        int mid = (lo + hi) >> 1;
        if (req_off[mid] <= t) lo = mid; else hi = mid;
    }
    const int32_t pos = (int32_t)(t - req_off[lo]);
    const int32_t delta = pos - cand[r];
    const int64_t page = block_table[(int64_t)lo * max_pages + pos / A.P];
    const int half = A.D / 2, chunks = half / 8, vvec = A.G * A.D / 8;
    const uint4 *src = in + r * (int64_t)A.L * 2 * vvec;
    for (int layer = layer_begin; layer < layer_end; ++layer) {
        const uint4 *sk = src + (layer * 2 + 0) * vvec;
        const uint4 *sv = src + (layer * 2 + 1) * vvec;
        uint4 *dk = reinterpret_cast<uint4 *>(A.row(page, layer, 0, pos % A.P));
        uint4 *dv = reinterpret_cast<uint4 *>(A.row(page, layer, 1, pos % A.P));
        for (int v = threadIdx.x; v < vvec; v += blockDim.x) dv[v] = sv[v];
        if (cos_t == nullptr || delta == 0) {
            for (int v = threadIdx.x; v < vvec; v += blockDim.x) dk[v] = sk[v];
        } else {
            for (int it = threadIdx.x; it < A.G * chunks; it += blockDim.x) {
                const int g = it / chunks, c = it % chunks;
                const int vlo = g * (A.D / 8) + c, vhi = vlo + chunks;
                uint4 lo_o, hi_o;
                rope8(sk[vlo], sk[vhi], lo_o, hi_o, cos_t, sin_t, delta, half, c);
                dk[vlo] = lo_o;
                dk[vhi] = hi_o;
            }
        }
    }
}

}  // namespace kvs

using namespace kvs;

// F3/F1 entry transfer (reference pool.py:100-123 insert, :174-241 KVSH
// save/load): an entry's K/V as dense fp32 [layer][token][kv_head][d_k] (the
// KVSH file order) <-> its arena pages (bf16, head dims in padded lanes:
// first half -> [0, d/2), second half -> [64, 64 + d/2)).  One CTA per
// (layer, token) row; both K and V.  Import rounds to bf16 (RNE) and zeroes
// the padding lanes; export widens exactly.
template <bool kImport>
__global__ void __launch_bounds__(128) entry_rows_kernel(Arena A, const int32_t *__restrict__ pages,
                                                         int64_t n, int32_t d_k, float *__restrict__ k,
                                                         float *__restrict__ v) {
    const int64_t row = blockIdx.x;                 // layer * n + token
    const int layer = (int)(row / n);
    const int64_t tok = row % n;
    const int64_t page = pages[tok / A.P];
    const int G = A.G;
    for (int kv = 0; kv < 2; ++kv) {
        __nv_bfloat16 *dst = A.row(page, layer, kv, (int)(tok % A.P));
        float *x = (kv == 0 ? k : v) + row * (int64_t)G * d_k;
        for (int e = threadIdx.x; e < G * A.D; e += blockDim.x) {
            const int g = e / A.D, lane = e % A.D;
            // which model dim sits in this lane (-1: padding)
            const int half = d_k / 2;
            const int d = lane < half ? lane : (lane >= 64 && lane < 64 + half ? half + lane - 64 : -1);
            if (kImport) {
                dst[e] = d >= 0 ? __float2bfloat16_rn(x[g * d_k + d]) : __float2bfloat16_rn(0.f);
            } else if (d >= 0) {
                x[g * d_k + d] = __bfloat162float(dst[e]);
            }
        }
    }
}

extern "C" {

static kvs_status gather_impl(const kvs_kv_arena *arena, const kvs_batch *batch,
                              const int32_t *src_slot, const int32_t *src_cand,
                              const int32_t *slot_pages, int32_t slot_max_pages,
                              const int32_t *slot_owner, const unsigned long long *peer_base,
                              int32_t layer_begin, int32_t layer_end, const kvs_rope *rope,
                              kvs_stream_t stream) {
    KVS_REQUIRE(arena && batch, KVS_EPARAM, "null arena/batch");
    KVS_REQUIRE(arena->head_dim % 16 == 0, KVS_ESHAPE, "head_dim must be a multiple of 16");
    KVS_REQUIRE(0 <= layer_begin && layer_begin <= layer_end && layer_end <= arena->num_layers,
                KVS_EPARAM, "bad layer range");
    KVS_REQUIRE((slot_owner == nullptr) == (peer_base == nullptr), KVS_EPARAM,
                "slot_owner and peer_base go together");
    if (batch->n_total <= 0 || layer_begin == layer_end) return KVS_OK;
    KVS_REQUIRE(batch->n_total < (1ll << 31), KVS_EPARAM, "batch too large");
    cudaStream_t s = (cudaStream_t)stream;
    gather_kv_kernel<<<(unsigned)batch->n_total, 128, 0, s>>>(
        make_arena(arena), batch->req_off, batch->n_req, batch->block_table, batch->max_pages,
        src_slot, src_cand, slot_pages, slot_max_pages, layer_begin, layer_end,
        rope ? rope->cos : nullptr, rope ? rope->sin : nullptr, slot_owner, peer_base);
    KVS_CHECK_LAUNCH("kvs_gather_kv");
    return KVS_OK;
}

kvs_status kvs_gather_kv(const kvs_kv_arena *arena, const kvs_batch *batch,
                         const int32_t *src_slot, const int32_t *src_cand,
                         const int32_t *slot_pages, int32_t slot_max_pages, int32_t layer_begin,
                         int32_t layer_end, const kvs_rope *rope, kvs_stream_t stream) {
    return gather_impl(arena, batch, src_slot, src_cand, slot_pages, slot_max_pages, nullptr,
                       nullptr, layer_begin, layer_end, rope, stream);
}

kvs_status kvs_gather_kv_peer(const kvs_kv_arena *arena, const kvs_batch *batch,
                              const int32_t *src_slot, const int32_t *src_cand,
                              const int32_t *slot_pages, int32_t slot_max_pages,
                              const int32_t *slot_owner, const uint64_t *peer_base,
                              int32_t layer_begin, int32_t layer_end, const kvs_rope *rope,
                              kvs_stream_t stream) {
    KVS_REQUIRE(slot_owner && peer_base, KVS_EPARAM, "null slot_owner/peer_base");
    return gather_impl(arena, batch, src_slot, src_cand, slot_pages, slot_max_pages, slot_owner,
                       reinterpret_cast<const unsigned long long *>(peer_base), layer_begin,
                       layer_end, rope, stream);
}

static kvs_status qkv_scatter_impl(const void *qkv, const int32_t *src_row, int64_t n_rows,
                                int32_t num_heads,
                                const int32_t *row_req, const int32_t *row_pos,
                                const uint8_t *write_kv, int32_t layer, const kvs_kv_arena *arena,
                                const kvs_batch *batch, const kvs_rope *rope, void *q_out,
                                void *k_out, void *v_out, kvs_stream_t stream) {
    KVS_REQUIRE(arena && batch, KVS_EPARAM, "null arena/batch");
    KVS_REQUIRE(arena->head_dim % 16 == 0, KVS_ESHAPE, "head_dim must be a multiple of 16");
    KVS_REQUIRE(num_heads % arena->kv_heads == 0, KVS_ESHAPE, "num_heads % kv_heads != 0");
    if (n_rows <= 0) return KVS_OK;
    cudaStream_t s = (cudaStream_t)stream;
    const size_t row_bytes = (size_t)((q_out != nullptr ? num_heads : 0) + 2 * arena->kv_heads) *
                             arena->head_dim * 2;
    const size_t smem = kScatSlots * row_bytes;
    if (arena->head_dim == 128 && smem <= 200 * 1024 && getenv("KVS_SCATTER_V1") == nullptr) {
        cudaFuncSetAttribute(qkv_scatter2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, qkv_scatter2_kernel, kScatThreads,
                                                      smem);
        const int64_t grid = std::min<int64_t>(n_rows, (int64_t)kNumSMs * std::max(per_sm, 1));
        qkv_scatter2_kernel<<<(unsigned)grid, kScatThreads, smem, s>>>(
            (const __nv_bfloat16 *)qkv, n_rows, num_heads, make_arena(arena), row_req, row_pos,
            write_kv, layer, batch->block_table, batch->max_pages, rope ? rope->cos : nullptr,
            rope ? rope->sin : nullptr, (__nv_bfloat16 *)q_out, (__nv_bfloat16 *)k_out,
            (__nv_bfloat16 *)v_out, src_row);
    } else {
        KVS_REQUIRE(src_row == nullptr, KVS_EPARAM,
                    "row-indexed scatter needs head_dim 128 (the TMA-ring kernel)");
        qkv_rope_scatter_kernel<<<(unsigned)n_rows, 256, 0, s>>>(
            (const __nv_bfloat16 *)qkv, num_heads, make_arena(arena), row_req, row_pos, write_kv,
            layer, batch->block_table, batch->max_pages, rope ? rope->cos : nullptr,
            rope ? rope->sin : nullptr, (__nv_bfloat16 *)q_out, (__nv_bfloat16 *)k_out,
            (__nv_bfloat16 *)v_out);
    }
    KVS_CHECK_LAUNCH("kvs_qkv_rope_scatter");
    return KVS_OK;
}

kvs_status kvs_qkv_rope_scatter(const void *qkv, int64_t n_rows, int32_t num_heads,
                                const int32_t *row_req, const int32_t *row_pos,
                                const uint8_t *write_kv, int32_t layer, const kvs_kv_arena *arena,
                                const kvs_batch *batch, const kvs_rope *rope, void *q_out,
                                void *k_out, void *v_out, kvs_stream_t stream) {
    return qkv_scatter_impl(qkv, nullptr, n_rows, num_heads, row_req, row_pos, write_kv, layer,
                            arena, batch, rope, q_out, k_out, v_out, stream);
}

kvs_status kvs_qkv_rope_scatter_rows(const void *qkv, const int32_t *src_row, int64_t n_rows,
                                     int32_t num_heads, const int32_t *row_req,
                                     const int32_t *row_pos, const uint8_t *write_kv,
                                     int32_t layer, const kvs_kv_arena *arena,
                                     const kvs_batch *batch, const kvs_rope *rope, void *q_out,
                                     void *k_out, void *v_out, kvs_stream_t stream) {
    KVS_REQUIRE(src_row != nullptr, KVS_EPARAM, "null src_row");
    return qkv_scatter_impl(qkv, src_row, n_rows, num_heads, row_req, row_pos, write_kv, layer,
                            arena, batch, rope, q_out, k_out, v_out, stream);
}

kvs_status kvs_embed_rows(const void *table, int64_t width, const int64_t *ids,
                          const int32_t *rows, int64_t n_rows, void *out, float *out_f32,
                          kvs_stream_t stream) {
    KVS_REQUIRE(width % 8 == 0, KVS_ESHAPE, "embedding width must be a multiple of 8");
    if (n_rows <= 0) return KVS_OK;
    embed_rows_kernel<<<(unsigned)n_rows, 128, 0, (cudaStream_t)stream>>>(
        (const __nv_bfloat16 *)table, width, ids, rows, (__nv_bfloat16 *)out, out_f32);
    KVS_CHECK_LAUNCH("kvs_embed_rows");
    return KVS_OK;
}

kvs_status kvs_build_rows(const int64_t *req_off, int32_t n_req, const int32_t *src_slot,
                          const uint8_t *selected, int32_t *counts, const int64_t *row_off,
                          int32_t *row_tok, int32_t *row_req, int32_t *row_pos, uint8_t *write_kv,
                          kvs_stream_t stream) {
    KVS_REQUIRE(n_req >= 1, KVS_EPARAM, "n_req must be >= 1");
    build_rows_kernel<<<n_req, 1024, 0, (cudaStream_t)stream>>>(
        req_off, src_slot, selected, counts, row_off, row_tok, row_req, row_pos, write_kv);
    KVS_CHECK_LAUNCH("kvs_build_rows");
    return KVS_OK;
}

kvs_status kvs_pack_rows(const kvs_kv_arena *arena, const int32_t *slot, const int32_t *cand,
                         int64_t n_rows, const int32_t *slot_pages, int32_t slot_max_pages,
                         void *out, kvs_stream_t stream) {
    KVS_REQUIRE(arena != nullptr, KVS_EPARAM, "null arena");
    KVS_REQUIRE((arena->kv_heads * arena->head_dim) % 8 == 0, KVS_ESHAPE, "row width % 8 != 0");
    if (n_rows <= 0) return KVS_OK;
    pack_rows_kernel<<<(unsigned)n_rows, 128, 0, (cudaStream_t)stream>>>(
        make_arena(arena), slot, cand, slot_pages, slot_max_pages, (uint4 *)out);
    KVS_CHECK_LAUNCH("kvs_pack_rows");
    return KVS_OK;
}

kvs_status kvs_unpack_rows(const kvs_kv_arena *arena, const kvs_batch *batch,
                           const int64_t *flat_t, const int32_t *cand, int64_t n_rows,
                           const void *in, const kvs_rope *rope, int32_t layer_begin,
                           int32_t layer_end, const uint8_t *skip, kvs_stream_t stream) {
    KVS_REQUIRE(arena && batch, KVS_EPARAM, "null arena/batch");
    KVS_REQUIRE(arena->head_dim % 16 == 0, KVS_ESHAPE, "head_dim must be a multiple of 16");
    KVS_REQUIRE(0 <= layer_begin && layer_begin <= layer_end && layer_end <= arena->num_layers,
                KVS_EPARAM, "layer range [%d, %d) outside [0, %d)", layer_begin, layer_end,
                arena->num_layers);
    if (n_rows <= 0 || layer_begin == layer_end) return KVS_OK;
    unpack_rows_kernel<<<(unsigned)n_rows, 128, 0, (cudaStream_t)stream>>>(
        make_arena(arena), batch->req_off, batch->n_req, batch->block_table, batch->max_pages,
        flat_t, cand, (const uint4 *)in, rope ? rope->cos : nullptr, rope ? rope->sin : nullptr,
        layer_begin, layer_end, skip);
    KVS_CHECK_LAUNCH("kvs_unpack_rows");
    return KVS_OK;
}

kvs_status kvs_entry_import(const kvs_kv_arena *arena, const int32_t *pages, int64_t n_tokens,
                            int32_t d_k, const float *k, const float *v, kvs_stream_t stream) {
    KVS_REQUIRE(arena != nullptr && pages != nullptr, KVS_EPARAM, "null arena/pages");
    KVS_REQUIRE(d_k >= 2 && d_k % 2 == 0 && d_k <= arena->head_dim, KVS_ESHAPE,
                "d_k must be even and <= head_dim");
    if (n_tokens <= 0) return KVS_OK;
    entry_rows_kernel<true><<<(unsigned)(n_tokens * arena->num_layers), 128, 0,
                              (cudaStream_t)stream>>>(make_arena(arena), pages, n_tokens, d_k,
                                                      const_cast<float *>(k), const_cast<float *>(v));
    KVS_CHECK_LAUNCH("kvs_entry_import");
    return KVS_OK;
}

kvs_status kvs_entry_export(const kvs_kv_arena *arena, const int32_t *pages, int64_t n_tokens,
                            int32_t d_k, float *k, float *v, kvs_stream_t stream) {
    KVS_REQUIRE(arena != nullptr && pages != nullptr, KVS_EPARAM, "null arena/pages");
    KVS_REQUIRE(d_k >= 2 && d_k % 2 == 0 && d_k <= arena->head_dim, KVS_ESHAPE,
                "d_k must be even and <= head_dim");
    if (n_tokens <= 0) return KVS_OK;
    entry_rows_kernel<false><<<(unsigned)(n_tokens * arena->num_layers), 128, 0,
                               (cudaStream_t)stream>>>(make_arena(arena), pages, n_tokens, d_k, k, v);
    KVS_CHECK_LAUNCH("kvs_entry_export");
    return KVS_OK;
}

}  // extern "C"
