// D3 decode-stage DHD as ONE fused, persistent, streaming kernel.
//
// select_decode_step (reference selection.py:80-105) for every request r of a
// decode batch: w_i = mean_h softmax_i(q_t[r,h] . K_i / sqrt(d)) over ALL
// ctx_len[r] rows of the probe layer (no mask), score_i = w_i * dvL1_i for the
// prefill rows (decode rows have zero deviation, engine.py:145-147), then the
// top min(n_extra, #eligible) eligible rows by (score desc, position asc)
// (selection.py:63-66), returned ascending; chosen rows leave `eligible`.
//
// The bound is HBM: every key row of every request is read once (kv_heads x
// 256 B at the probe layer).  One cooperative launch of one CTA per SM:
//
// phase 1, streaming.  Work items are (request, 64-key page, kv head): 16 KB
// of K plus the group's query heads, handed out one at a time from a global
// ticket to whichever of the CTAs' 6 warps is ready (faster SMs take more).
// Every warp keeps two of its own items in flight (SWIZZLE_128B TMA loads
// with an L2 evict-first hint, one mbarrier per stage, no producer warp, so
// no warp waits behind another's stage); the next ticket and its arena page
// are fetched one item ahead.
// Q.K^T runs on the tensor cores (mma.sync m16n8k16 bf16 -> fp32; A = the
// swizzled K tile through conflict-free ldmatrix, B = the group's <= 8 query
// heads from the same stage), and the epilogue writes the logits (log2
// domain, key-major, L2-resident) and per-(page, head) softmax partials.
//
// grid barrier.  Before arriving, each CTA already compacts the row list of
// its first phase-2 unit (eligibility and dv-L1 of those rows) - nothing
// phase 1 writes is needed for that.
//
// phase 2, selection.  Units are (request, key slice), slices sized so every
// CTA has one when the batch is smaller than the grid.  Per unit: the page
// partials and the listed rows' logits are gathered into shared memory with
// cp.async in one round trip, per-head statistics are folded, the rows are
// scored warp-cooperatively from shared memory into register top-n_extra
// lists, a block merge gives the slice's candidates, and the last slice of a
// request (release/acquire counter) merges the slices and writes chosen /
// n_chosen / eligible.  Counters and the barrier reset themselves.
//
// Measured on one B200 (tools/micro_d3.py, profiles/r2_d3_*): 0.62 / 0.67 /
// 0.68 of HBM at 64 / 128 / 256 requests x 4096 context; pure streaming
// with this access pattern reaches 0.80-0.98, the rest is phase 2's latency
// chain (~25 us: barrier, gather, fold, scoring, merges).
#include "common.cuh"

namespace kvs {
namespace d3 {

constexpr int kWarps = 6;              // every warp streams its own items (no producer warp)
constexpr int kThreads = 32 * kWarps;
constexpr int kBuf = 2;                // stages per warp: the next item loads under this one
constexpr int kKBytes = 16384;         // 64 keys x 128 dims bf16 (two 8 KB halves)
constexpr int kStageBytes = kKBytes + 2048;   // + the group's query heads (two 1 KB halves)
constexpr int kTileKeys = 64;
constexpr int kMaxReq = 1024;
constexpr int kMaxK = 16;              // n_extra supported by the fused kernel
constexpr int kMaxHeads = 64;

struct Smem {
    alignas(1024) uint8_t ring[kWarps][kBuf][kStageBytes];   // phase 2: scratch
    uint64_t full[kWarps][kBuf];
    int32_t item_off[kMaxReq + 1];
    int32_t chunk_sum[kThreads];
    float hm[kMaxHeads], hz[kMaxHeads];
    uint64_t red[kThreads / 32];
    uint64_t wkeys[kThreads / 32][32];
    int32_t flag, n_list;
};

__device__ __forceinline__ void ldmatrix_x4(uint32_t addr, uint32_t &a0, uint32_t &a1,
                                            uint32_t &a2, uint32_t &a3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
                 : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3)
                 : "r"(addr));
}

__device__ __forceinline__ void mma_bf16_16816(float *c, uint32_t a0, uint32_t a1, uint32_t a2,
                                               uint32_t a3, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 "
        "{%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, {%0, %1, %2, %3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// K rows are streamed exactly once: L2 evict-first, so the logits and page
// partials written alongside stay in L2 for phase 2
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void tma_load_4d_stream(void *dst, const CUtensorMap *map, uint64_t *bar,
                                                   int c0, int c1, int c2, int c3, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%3, %4, %5, %6}], [%2], %7;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2),
        "r"(c3), "l"(pol)
        : "memory");
}

__device__ __forceinline__ int ld_acquire(const int32_t *p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

#ifdef KVS_D3_TRACE
__device__ unsigned long long g_trace[kNumSMs][8];
#define D3_STAMP(i)                                                                  \
    do {                                                                             \
        if (threadIdx.x == 0 && blockIdx.x < kNumSMs) {                              \
            unsigned long long t;                                                    \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));                    \
            g_trace[blockIdx.x][i] = t;                                              \
        }                                                                            \
    } while (0)
#else
#define D3_STAMP(i) do {} while (0)
#endif

struct Params {
    int32_t H, G, HQ;
    const int32_t *ctx_len;
    int32_t n_req, max_ctx, layer, num_layers;
    const int32_t *block_table;
    int32_t max_pages;
    float scale_log2;
    const float *dv_l1;
    uint8_t *eligible;
    const int64_t *req_off;
    int32_t n_extra;
    int32_t *chosen, *n_chosen;
    float *scores_out;
    float *logits;           // [n_req][ld][Hp] (key-major, heads padded to 4)
    float2 *part;            // [n_req][tiles][H] per-page (max, sum exp2)
    uint64_t *cand;          // [n_req][slices][kMaxK] per-slice top keys
    int32_t *ctr;            // [3 + n_req]: item ticket, barrier, exits, per-request slices done
    int32_t ld, tiles, Hp;
};

// (score desc, position asc) as an ascending 64-bit key
__device__ __forceinline__ uint64_t sel_key(float v, int i) {
    return ((uint64_t)(~__float_as_uint(fmaxf(v, 0.f))) << 32) | (uint32_t)i;
}

__device__ __forceinline__ uint64_t block_min(uint64_t v, Smem &sm) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const uint64_t x = __shfl_xor_sync(0xffffffffu, v, o);
        v = x < v ? x : v;
    }
    __syncthreads();
    if (lane == 0) sm.red[w] = v;
    __syncthreads();
    uint64_t b = sm.red[0];
#pragma unroll
    for (int k = 1; k < kThreads / 32; ++k) b = sm.red[k] < b ? sm.red[k] : b;
    return b;
}

// ---------------------------------------------------------------- phase 2
// Shared-memory layout of phase 2 (the phase-1 ring is free by then):
//   [0, 16 KB)     row list of the current chunk (position | eligible << 31)
//   [16, 32 KB)    the listed rows' dv-L1
//   [32, 64 KB)    page partials of the request (head statistics)
//   [64 KB, end)   the listed rows' logits, gathered with cp.async
constexpr int kListCap = 4096;
constexpr int kDvOff = kListCap * 4;
constexpr int kPartOff = 32 * 1024;
constexpr int kPartBytes = 32 * 1024;
constexpr int kLogitOff = 64 * 1024;

__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}

// Rows [i0, i1) of request r to score: the eligible rows, or with a scores
// output every prefill row (decode rows get score 0 right here).  Every
// eligibility byte and dv-L1 value is loaded with the list built.  Returns
// the count.
__device__ int build_list(const Params &p, Smem &sm, int64_t s, int lim, int i0, int i1,
                          float *scr) {
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    int32_t *list = reinterpret_cast<int32_t *>(&sm.ring[0][0][0]);
    float *dvl = reinterpret_cast<float *>(&sm.ring[0][0][0] + kDvOff);
    if (tid == 0) sm.n_list = 0;
    __syncthreads();
    const int lim_b = min(i1, lim);
    constexpr int kU = 12;                                       // loads in flight per thread
    for (int c0 = i0 + w * 32; c0 < i1; c0 += kU * kThreads) {   // warp-uniform trip count
        bool take[kU], el[kU];
        float dv[kU];
#pragma unroll
        for (int c = 0; c < kU; ++c) {
            const int i = c0 + c * kThreads + lane;
            el[c] = i < lim_b && p.eligible[s + i];
        }
#pragma unroll
        for (int c = 0; c < kU; ++c) {
            const int i = c0 + c * kThreads + lane;
            take[c] = i < lim_b && (scr || el[c]);
            dv[c] = i < lim_b ? p.dv_l1[s + i] : 0.f;
        }
#pragma unroll
        for (int c = 0; c < kU; ++c) {
            const int i = c0 + c * kThreads + lane;
            const unsigned m = __ballot_sync(0xffffffffu, take[c]);
            int base = 0;
            if (lane == 0 && m) base = atomicAdd(&sm.n_list, __popc(m));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (take[c]) {
                const int at = base + __popc(m & ((1u << lane) - 1));
                list[at] = i | (el[c] ? (int)0x80000000u : 0);
                dvl[at] = dv[c];
            }
            if (scr && i >= lim_b && i < i1) scr[i] = 0.f;       // decode rows score 0
        }
    }
    __syncthreads();
    return sm.n_list;
}

// cp.async gather of the logits rows list[j0, j0 + nb) into the staging area
// (Hp floats per row, 16-byte pieces spread over the CTA; nothing is held in
// registers, so every piece of the batch is in flight at once).
__device__ void gather_rows(const Params &p, Smem &sm, int r, int j0, int nb) {
    const int32_t *list = reinterpret_cast<const int32_t *>(&sm.ring[0][0][0]);
    const float *lg = p.logits + (int64_t)r * p.ld * p.Hp;
    const uint32_t dst = smem_u32(&sm.ring[0][0][0] + kLogitOff);
    const int nh4 = p.Hp >> 2;
    for (int e = threadIdx.x; e < nb * nh4; e += kThreads) {
        const int j = e / nh4, h4 = e - j * nh4;
        const int row = list[j0 + j] & 0x7fffffff;
        cp_async16(dst + (uint32_t)(j * p.Hp + 4 * h4) * 4u, lg + (int64_t)row * p.Hp + 4 * h4);
    }
}

// cp.async of the page partials of tiles [t0, t0 + nt) of request r.
__device__ void gather_part(const Params &p, Smem &sm, int r, int t0, int nt) {
    const float2 *src = p.part + ((int64_t)r * p.tiles + t0) * p.H;
    const uint32_t dst = smem_u32(&sm.ring[0][0][0] + kPartOff);
    const int n16 = (nt * p.H * 8 + 15) / 16;                 // 16-byte pieces (H*8 is 16-aligned
    for (int e = threadIdx.x; e < n16; e += kThreads)          //  for even H; odd H reads a pad)
        cp_async16(dst + e * 16u, reinterpret_cast<const uint8_t *>(src) + e * 16);
}

// Fold the staged partials of nt tiles into the per-head running (hm, hz).
__device__ void fold_part(const Params &p, Smem &sm, int nt) {
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const float2 *stage = reinterpret_cast<const float2 *>(&sm.ring[0][0][0] + kPartOff);
    for (int h = w; h < p.H; h += kThreads / 32) {
        float m = -INFINITY, z = 0.f;
        for (int t = lane; t < nt; t += 32) {
            const float2 pz = stage[t * p.H + h];
            if (pz.x == -INFINITY) continue;
            const float mn = fmaxf(m, pz.x);
            z = z * fast_exp2(m - mn) + pz.y * fast_exp2(pz.x - mn);
            m = mn;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const float mo = __shfl_xor_sync(0xffffffffu, m, o);
            const float zo = __shfl_xor_sync(0xffffffffu, z, o);
            const float mn = fmaxf(m, mo);
            z = (m == -INFINITY ? 0.f : z * fast_exp2(m - mn)) +
                (mo == -INFINITY ? 0.f : zo * fast_exp2(mo - mn));
            m = mn;
        }
        if (lane == 0 && m != -INFINITY) {
            const float m0 = sm.hm[h];
            const float mn = fmaxf(m0, m);
            sm.hz[h] = (m0 == -INFINITY ? 0.f : sm.hz[h] * fast_exp2(m0 - mn)) +
                       z * fast_exp2(m - mn);
            sm.hm[h] = mn;
        }
    }
}

// Scores of the staged rows list[j0, j0 + nb), warp-cooperative from shared
// memory: 8 lanes read one row's Hp logits (16-byte pieces), 4 rows per warp
// instruction, kGroups groups of 4 rows per warp; the 8-lane partial sums
// meet by xor shuffles, the group's first lane forms the row's selection
// key, and the warp's keys are spread over all lanes for the register top-KM.
template <int KM>
__device__ void score_rows(const Params &p, Smem &sm, int j0, int nb, float *scr,
                           uint64_t *top) {
    constexpr int kGroups = 8;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int32_t *list = reinterpret_cast<const int32_t *>(&sm.ring[0][0][0]);
    const float *dvl = reinterpret_cast<const float *>(&sm.ring[0][0][0] + kDvOff);
    const float *stg = reinterpret_cast<const float *>(&sm.ring[0][0][0] + kLogitOff);
    const float invH = 1.f / (float)p.H;
    const int nh4 = p.Hp >> 2;
    const int sub = lane >> 3, h4l = lane & 7;
    uint64_t *wk = sm.wkeys[w];
    for (int b0 = w * 4 * kGroups; b0 < nb; b0 += 4 * kGroups * (kThreads / 32)) {
        float wsum[kGroups];
#pragma unroll
        for (int q = 0; q < kGroups; ++q) wsum[q] = 0.f;
        for (int hb = 0; hb < nh4; hb += 8) {
            const int h4 = hb + h4l;
            if (h4 < nh4) {
                float hm[4], hz[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int h = 4 * h4 + e;
                    hm[e] = h < p.H ? sm.hm[h] : 0.f;
                    hz[e] = h < p.H ? sm.hz[h] : 0.f;
                }
#pragma unroll
                for (int q = 0; q < kGroups; ++q) {
                    const int j = b0 + 4 * q + sub;
                    if (j < nb) {
                        const float4 x = *reinterpret_cast<const float4 *>(stg + j * p.Hp + 4 * h4);
                        wsum[q] += fast_exp2(x.x - hm[0]) * hz[0] + fast_exp2(x.y - hm[1]) * hz[1] +
                                   fast_exp2(x.z - hm[2]) * hz[2] + fast_exp2(x.w - hm[3]) * hz[3];
                    }
                }
            }
        }
#pragma unroll
        for (int q = 0; q < kGroups; ++q) {
#pragma unroll
            for (int o = 1; o < 8; o <<= 1) wsum[q] += __shfl_xor_sync(0xffffffffu, wsum[q], o);
            const int j = b0 + 4 * q + sub;
            if (h4l == 0) {
                uint64_t key = ~0ull;
                if (j < nb) {
                    const int li = list[j0 + j];
                    const int row = li & 0x7fffffff;
                    const float v = wsum[q] * invH * dvl[j0 + j];
                    if (scr) scr[row] = v;
                    if (li < 0) key = sel_key(v, row);              // eligible bit set
                }
                wk[4 * q + sub] = key;
            }
        }
        __syncwarp();
        {
            uint64_t key = wk[lane];
            if (key < top[KM - 1]) {
#pragma unroll
                for (int jj = 0; jj < KM; ++jj)
                    if (key < top[jj]) {
                        const uint64_t t = top[jj];
                        top[jj] = key;
                        key = t;
                    }
            }
        }
        __syncwarp();
    }
}

// Phase 2, one (request, key slice): head statistics, the scores of the
// slice's rows (in list chunks; the first chunk may have been built before
// the grid barrier), the slice's top-n_extra eligible rows; the request's
// last slice merges.  prebuilt: row count of a list already in shared
// memory for the slice's first chunk, or -1.  The first logits batch and the
// first partials chunk are gathered together (one memory round trip).
template <int KM>
__device__ void finish_slice(const Params &p, Smem &sm, int r, int slice, int n_slices,
                             int prebuilt) {
    const int tid = threadIdx.x;
    const int n = p.ctx_len[r];
    const int64_t s = p.req_off[r];
    const int n_pre = (int)(p.req_off[r + 1] - s);
    const int lim = n_pre < n ? n_pre : n;
    const int K = p.n_extra;
    const int T = (n + kTileKeys - 1) / kTileKeys;
    const int tcap = kPartBytes / (p.H * 8);
    const int rcap = (int)((sizeof(sm.ring) - kLogitOff) / (p.Hp * 4));   // rows per batch
    uint64_t top[KM];
#pragma unroll
    for (int j = 0; j < KM; ++j) top[j] = ~0ull;
    float *scr = p.scores_out ? p.scores_out + (int64_t)r * p.max_ctx : nullptr;
    const int per = (n + n_slices - 1) / n_slices;
    const int a = slice * per, b = min(n, a + per);
    for (int h = tid; h < p.H; h += kThreads) {
        sm.hm[h] = -INFINITY;
        sm.hz[h] = 0.f;
    }
    bool first = true;
    for (int c0 = a; c0 < b || first; c0 += kListCap) {
        const int nl = c0 >= b ? 0 : (c0 == a && prebuilt >= 0)
                                         ? prebuilt
                                         : build_list(p, sm, s, lim, c0, min(b, c0 + kListCap), scr);
        D3_STAMP(3);
        for (int j0 = 0; j0 < nl || first; j0 += rcap) {
            const int nb = min(rcap, nl - j0);
            if (nb > 0) gather_rows(p, sm, r, j0, nb);
            if (first) {
                // head statistics: the partials' first chunk rides with the rows
                for (int t0 = 0; t0 < T; t0 += tcap) {
                    const int nt = min(tcap, T - t0);
                    gather_part(p, sm, r, t0, nt);
                    cp_async_wait_all();
                    __syncthreads();
                    fold_part(p, sm, nt);
                    __syncthreads();
                }
                for (int h = tid; h < p.H; h += kThreads) sm.hz[h] = 1.f / sm.hz[h];
                first = false;
                D3_STAMP(2);
            }
            cp_async_wait_all();
            __syncthreads();
            D3_STAMP(4);
            if (nb > 0) score_rows<KM>(p, sm, j0, nb, scr, top);
            __syncthreads();                               // staging reused next
        }
    }
    // keep only the first K of each list (KM may exceed n_extra)
#pragma unroll
    for (int jj = 0; jj < KM; ++jj)
        if (jj >= K) top[jj] = ~0ull;
    D3_STAMP(5);
    uint64_t *cand = p.cand + ((int64_t)r * gridDim.x + slice) * kMaxK;
    for (int k = 0; k < K; ++k) {
        const uint64_t best = block_min(top[0], sm);
        if (best != ~0ull && top[0] == best) {             // keys are unique: one owner
#pragma unroll
            for (int j = 0; j + 1 < KM; ++j) top[j] = top[j + 1];
            top[KM - 1] = ~0ull;
        }
        if (tid == 0) cand[k] = best;
    }
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        sm.flag = atomicAdd(&p.ctr[3 + r], 1) == n_slices - 1;
        __threadfence();
    }
    __syncthreads();
    if (!sm.flag) return;
    D3_STAMP(6);
    // merge: n_slices sorted lists of K, staged in shared memory with one
    // round trip; thread t owns lists t, t + kThreads
    uint64_t *cs = reinterpret_cast<uint64_t *>(&sm.ring[0][0][0]);
    const uint64_t *all = p.cand + (int64_t)r * gridDim.x * kMaxK;
    for (int e = tid; e < n_slices * K; e += kThreads) {
        const int l = e / K, k = e - l * K;
        cs[e] = __ldcg(all + (int64_t)l * kMaxK + k);
    }
    __syncthreads();
    int ptr0 = 0, ptr1 = 0;
    int picked = 0;
    int32_t *out = p.chosen + (int64_t)r * K;
    int32_t *pick = reinterpret_cast<int32_t *>(cs + n_slices * K);
    for (int k = 0; k < K; ++k) {
        const int l0 = tid, l1 = tid + kThreads;
        const uint64_t x0 = l0 < n_slices && ptr0 < K ? cs[l0 * K + ptr0] : ~0ull;
        const uint64_t x1 = l1 < n_slices && ptr1 < K ? cs[l1 * K + ptr1] : ~0ull;
        const uint64_t mine = x0 < x1 ? x0 : x1;
        const uint64_t best = block_min(mine, sm);
        if (best == ~0ull) break;
        if (x0 == best) ++ptr0;
        else if (x1 == best) ++ptr1;
        if (tid == 0) pick[picked] = (int32_t)(best & 0xffffffffu);
        ++picked;
    }
    __syncthreads();
    if (tid == 0) {
        for (int x = 1; x < picked; ++x)                      // ascending (selection.py:66)
            for (int y = x; y > 0 && pick[y - 1] > pick[y]; --y) {
                const int32_t t = pick[y];
                pick[y] = pick[y - 1];
                pick[y - 1] = t;
            }
        for (int k = 0; k < K; ++k) {
            out[k] = k < picked ? pick[k] : -1;
            if (k < picked) p.eligible[s + pick[k]] = 0;
        }
        p.n_chosen[r] = picked;
        p.ctr[3 + r] = 0;                                    // ready for the next call
    }
    D3_STAMP(7);
}

template <int KM>
__global__ void __launch_bounds__(kThreads, 1)
    decode_select_fused_kernel(const __grid_constant__ CUtensorMap map_kv,
                               const __grid_constant__ CUtensorMap map_q, const Params p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1 KB-aligned view of dynamic shared memory (SWIZZLE_128B destinations);
    // pointer arithmetic on the shared array keeps the accesses LDS/STS
    Smem &sm = *reinterpret_cast<Smem *>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // ---- item offsets: items_r = pages(ctx_r) x kv_heads (block scan)
    {
        const int per = (p.n_req + kThreads - 1) / kThreads;
        const int a = tid * per, b = min(p.n_req, a + per);
        int sum = 0;
        for (int r = a; r < b; ++r) sum += ((p.ctx_len[r] + kTileKeys - 1) / kTileKeys) * p.G;
        sm.chunk_sum[tid] = sum;
        __syncthreads();
        if (tid == 0) {
            int acc = 0;
            for (int t = 0; t < kThreads; ++t) {
                const int x = sm.chunk_sum[t];
                sm.chunk_sum[t] = acc;
                acc += x;
            }
            sm.item_off[p.n_req] = acc;
            for (int w = 0; w < kWarps; ++w)
                for (int j = 0; j < kBuf; ++j) mbar_init(&sm.full[w][j], 1);
            fence_barrier_init();
        }
        __syncthreads();
        int acc = sm.chunk_sum[tid];
        for (int r = a; r < b; ++r) {
            sm.item_off[r] = acc;
            acc += ((p.ctx_len[r] + kTileKeys - 1) / kTileKeys) * p.G;
        }
        __syncthreads();
    }
    const int total = sm.item_off[p.n_req];
    const uint32_t qbytes = 2u * (uint32_t)p.HQ * 128u;
    // ---------------------------------------------------- phase 1: streaming
    // Items (request, page, kv head) are handed out one at a time from a
    // global ticket (ctr[0]) to whichever warp is ready, so SMs that stream
    // slower simply take fewer items (a static page split left the slowest
    // CTA finishing 20-60 us after the median).  A warp's tickets only grow,
    // so its request cursors move forward.  Lane 0 keeps the next two
    // tickets and the arena page of the first, so neither the ticket atomic
    // nor the block-table load sits in front of a TMA issue.
    const uint64_t pol = l2_evict_first_policy();
    int r_iss = 0, r_con = 0, r_pf = 0;
    auto advance = [&](int &r, int it) {
        while (sm.item_off[r + 1] <= it) ++r;
        return r;
    };
    auto page_of = [&](int it) -> int {
        if (it >= total) return 0;
        const int rl = advance(r_pf, it);
        return __ldg(p.block_table + (int64_t)rl * p.max_pages + (it - sm.item_off[rl]) / p.G);
    };
    int t_a = 0, t_b = 0, pg_a = 0, held[kBuf];
    if (lane == 0) {
        t_a = atomicAdd(&p.ctr[0], 1);
        t_b = atomicAdd(&p.ctr[0], 1);
        pg_a = page_of(t_a);
    }
    auto issue = [&](int buf) {                   // lane 0: the warp's next ticket into buf
        if (lane != 0) return;
        const int it = t_a, page = pg_a;
#pragma unroll
        for (int q = 0; q < kBuf; ++q)
            if (q == buf) held[q] = it;
        t_a = t_b;
        pg_a = page_of(t_a);
        t_b = t_a < total ? atomicAdd(&p.ctr[0], 1) : total;
        if (it >= total) return;
        const int r = advance(r_iss, it);
        const int rel = it - sm.item_off[r];
        const int g = rel % p.G;
        const int c3 = (page * p.num_layers + p.layer) * 2;          // K of the layer
        uint8_t *st = sm.ring[warp][buf];
        uint64_t *bar = &sm.full[warp][buf];
        fence_proxy_async_smem();
        mbar_expect_tx(bar, kKBytes + qbytes);
        tma_load_4d_stream(st, &map_kv, bar, 0, g, 0, c3, pol);
        tma_load_4d_stream(st + 8192, &map_kv, bar, 64, g, 0, c3, pol);
        tma_load_3d(st + kKBytes, &map_q, bar, 0, g * p.HQ, r);
        tma_load_3d(st + kKBytes + 1024, &map_q, bar, 64, g * p.HQ, r);
    };
    if (warp == 0 && lane == 0) {
        tma_prefetch(&map_kv);
        tma_prefetch(&map_q);
    }
#pragma unroll
    for (int j = 0; j < kBuf; ++j) issue(j);
    __syncwarp();
    for (int j = 0;; ++j) {
        const int buf = j % kBuf;
        int mine = 0;
#pragma unroll
        for (int q = 0; q < kBuf; ++q)
            if (q == buf) mine = held[q];
        const int it = __shfl_sync(0xffffffffu, mine, 0);
        if (it >= total) break;
        mbar_wait(&sm.full[warp][buf], (j / kBuf) & 1);
        const int r = advance(r_con, it);
        const int rel = it - sm.item_off[r];
        const int tile = rel / p.G, g = rel - tile * p.G;
        const int n = p.ctx_len[r];
        const uint32_t base = smem_u32(sm.ring[warp][buf]);
        float acc[4][4];
        // B (dims x heads, "col"): ldmatrix rows = heads (128-B swizzled rows)
        uint32_t qb[8][2];
        {
            const int hr = lane & 7, mi = lane >> 3;
#pragma unroll
            for (int kp = 0; kp < 4; ++kp) {                 // two k-steps per x4
                const int chunk = kp * 4 + mi;               // 16-byte chunk of 16 in a row
                const uint32_t addr = base + kKBytes + (chunk >> 3) * 1024 + hr * 128 +
                                      (((chunk & 7) ^ hr) << 4);
                ldmatrix_x4(addr, qb[2 * kp][0], qb[2 * kp][1], qb[2 * kp + 1][0],
                            qb[2 * kp + 1][1]);
            }
        }
        // a whole 64-key page of one kv head: 4 M tiles of 16 keys x <= 8 heads
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) {
#pragma unroll
            for (int e = 0; e < 4; ++e) acc[mt][e] = 0.f;
            const int jj = lane >> 3;
            const int row = mt * 16 + (jj & 1) * 8 + (lane & 7);
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
                const int chunk = ks * 2 + (jj >> 1);
                const uint32_t addr = base + (chunk >> 3) * 8192 + row * 128 +
                                      (((chunk & 7) ^ (row & 7)) << 4);
                uint32_t a0, a1, a2, a3;
                ldmatrix_x4(addr, a0, a1, a2, a3);
                mma_bf16_16816(acc[mt], a0, a1, a2, a3, qb[ks][0], qb[ks][1]);
            }
        }
        __syncwarp();
        // the stage is free again: this warp's item two ahead loads under the epilogue
        issue(buf);
        // epilogue: key rows 16mt + lane/4 (+8), head columns 2(lane%4) + {0,1}
        const int col = 2 * (lane & 3);
        const int kb = tile * kTileKeys + (lane >> 2);
        float *lg = p.logits + (int64_t)r * p.ld * p.Hp + g * p.HQ;
        float m[2] = {-INFINITY, -INFINITY};
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int key = kb + mt * 16 + (e >> 1) * 8;
                const float x = key < n ? acc[mt][e] * p.scale_log2 : -INFINITY;
                acc[mt][e] = x;
                m[e & 1] = fmaxf(m[e & 1], x);
                if (!(p.HQ & 1)) {
                    if ((e & 1) && key < n && col < p.HQ)     // even groups: one 8-byte store
                        *reinterpret_cast<float2 *>(lg + (int64_t)key * p.Hp + col) =
                            make_float2(acc[mt][e - 1], x);
                } else if (key < n && col + (e & 1) < p.HQ) {
                    lg[(int64_t)key * p.Hp + col + (e & 1)] = x;
                }
            }
#pragma unroll
        for (int c = 0; c < 2; ++c) {
#pragma unroll
            for (int o = 4; o < 32; o <<= 1)
                m[c] = fmaxf(m[c], __shfl_xor_sync(0xffffffffu, m[c], o));
            float z = 0.f;
            if (m[c] != -INFINITY)
#pragma unroll
                for (int mt = 0; mt < 4; ++mt)
                    z += fast_exp2(acc[mt][c] - m[c]) + fast_exp2(acc[mt][2 + c] - m[c]);
#pragma unroll
            for (int o = 4; o < 32; o <<= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
            if (lane < 4 && col + c < p.HQ)
                p.part[((int64_t)r * p.tiles + tile) * p.H + g * p.HQ + col + c] =
                    make_float2(m[c], z);
        }
    }
    // ---- phase 2 units: (request, key slice) per CTA
    const int G2 = gridDim.x;
    const int spr = p.n_req >= G2 ? 1 : G2 / p.n_req;         // slices per request
    const int n_units = p.n_req >= G2 ? p.n_req : p.n_req * spr;
    // the first unit's row list depends on nothing phase 1 writes: build it
    // while the slower CTAs are still streaming
    __syncthreads();                                           // ring free
    D3_STAMP(0);
    int prebuilt = -1;
    if ((int)blockIdx.x < n_units) {
        const int r = blockIdx.x / spr, slice = blockIdx.x % spr;
        const int n = p.ctx_len[r];
        if (n > 0) {
            const int64_t s0 = p.req_off[r];
            const int n_pre = (int)(p.req_off[r + 1] - s0);
            const int per = (n + spr - 1) / spr;
            const int a = slice * per, b = min(n, a + per);
            float *scr = p.scores_out ? p.scores_out + (int64_t)r * p.max_ctx : nullptr;
            if (a < b) prebuilt = build_list(p, sm, s0, min(n_pre, n), a, min(b, a + kListCap), scr);
        }
    }
    // ---- grid barrier (cooperative launch: every CTA is resident)
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        atomicAdd(&p.ctr[1], 1);
        while (ld_acquire(&p.ctr[1]) < (int)gridDim.x) __nanosleep(64);
    }
    __syncthreads();
    D3_STAMP(1);
    for (int u = blockIdx.x; u < n_units; u += G2) {
        const int r = u / spr, slice = u % spr;
        if (p.ctx_len[r] <= 0) {
            if (slice == 0 && tid == 0) {
                for (int k = 0; k < p.n_extra; ++k) p.chosen[(int64_t)r * p.n_extra + k] = -1;
                p.n_chosen[r] = 0;
            }
            continue;
        }
        finish_slice<KM>(p, sm, r, slice, spr, u == (int)blockIdx.x ? prebuilt : -1);
        __syncthreads();
    }
    // the last CTA out resets the work ticket and the barrier
    if (tid == 0 && atomicAdd(&p.ctr[2], 1) == G2 - 1) {
        p.ctr[0] = 0;
        p.ctr[1] = 0;
        p.ctr[2] = 0;
    }
}

}  // namespace d3

#ifdef KVS_D3_TRACE
extern "C" void kvs_d3_trace(unsigned long long *out) {
    cudaMemcpyFromSymbol(out, d3::g_trace, sizeof(d3::g_trace));
}
#endif

static inline size_t al256(size_t x) { return (x + 255) & ~(size_t)255; }

// The counter header (work ticket, grid barrier, exits, per-request slice
// counters) has one fixed size for every n_req, and the two-kernel fallback
// lays its buffers out after it too: a workspace reused across calls of any
// shape or path keeps the header zero between calls.
size_t d3_counter_bytes() { return al256(sizeof(int32_t) * ((size_t)d3::kMaxReq + 3)); }

size_t d3_fused_workspace(int32_t n_req, int32_t num_heads, int32_t max_ctx) {
    const size_t ld = ((size_t)max_ctx + 3) & ~(size_t)3;
    const size_t tiles = ((size_t)max_ctx + d3::kTileKeys - 1) / d3::kTileKeys;
    const size_t hp = ((size_t)num_heads + 3) & ~(size_t)3;
    return d3_counter_bytes() +
           al256(sizeof(float) * (size_t)n_req * hp * ld) +
           al256(sizeof(float2) * (size_t)n_req * tiles * num_heads + 16) +
           al256(sizeof(uint64_t) * (size_t)n_req * 2 * kNumSMs * d3::kMaxK);
}

bool d3_fused_supported(const kvs_kv_arena *arena, int32_t n_req, int32_t num_heads,
                        int32_t n_extra) {
    return arena->page_size == d3::kTileKeys && arena->head_dim == 128 &&
           num_heads <= d3::kMaxHeads && num_heads % 2 == 0 &&
           num_heads / arena->kv_heads <= 8 &&
           n_extra >= 1 && n_extra <= d3::kMaxK && n_req >= 1 && n_req <= d3::kMaxReq;
}

kvs_status d3_fused_launch(const void *q_t, int32_t num_heads, const int32_t *ctx_len,
                           int32_t max_ctx, const float *dv_l1, uint8_t *eligible, int32_t layer,
                           const kvs_kv_arena *arena, const kvs_batch *batch, int32_t n_extra,
                           float softmax_scale, int32_t *chosen, int32_t *n_chosen, float *scores,
                           void *ws, cudaStream_t s) {
    CUtensorMap map_kv, map_q;
    KVS_REQUIRE(make_kv_map(&map_kv, arena), KVS_ECUDA, "KV tensor map");
    const int hq = num_heads / arena->kv_heads;
    {
        // q_t [n_req][H][128] bf16; box = 64 dims x the group's hq heads x 1 request
        uint64_t dims[3] = {128, (uint64_t)num_heads, (uint64_t)batch->n_req};
        uint64_t strides[2] = {256, (uint64_t)num_heads * 256};
        uint32_t box[3] = {64, (uint32_t)hq, 1};
        KVS_REQUIRE(encode_tmap(&map_q, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(q_t),
                                dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B),
                    KVS_ECUDA, "q tensor map");
    }
    d3::Params p;
    p.H = num_heads;
    p.G = arena->kv_heads;
    p.HQ = hq;
    p.ctx_len = ctx_len;
    p.n_req = batch->n_req;
    p.max_ctx = max_ctx;
    p.layer = layer;
    p.num_layers = arena->num_layers;
    p.block_table = batch->block_table;
    p.max_pages = batch->max_pages;
    p.scale_log2 = softmax_scale * 1.4426950408889634f;
    p.dv_l1 = dv_l1;
    p.eligible = eligible;
    p.req_off = batch->req_off;
    p.n_extra = n_extra;
    p.chosen = chosen;
    p.n_chosen = n_chosen;
    p.scores_out = scores;
    p.ld = (max_ctx + 3) & ~3;
    p.tiles = (max_ctx + d3::kTileKeys - 1) / d3::kTileKeys;
    p.Hp = (num_heads + 3) & ~3;
    char *w = (char *)ws;
    p.ctr = (int32_t *)w;
    w += d3_counter_bytes();
    p.logits = (float *)w;
    w += al256(sizeof(float) * (size_t)batch->n_req * p.Hp * p.ld);
    p.part = (float2 *)w;
    w += al256(sizeof(float2) * (size_t)batch->n_req * p.tiles * num_heads + 16);
    p.cand = (uint64_t *)w;
    const int smem = (int)sizeof(d3::Smem) + 1024;
    // the per-thread top-n_extra list lives in registers: a 4-entry kernel for
    // the paper's n_extra <= 4, a 16-entry one above
    const void *fn = n_extra <= 4 ? (const void *)d3::decode_select_fused_kernel<4>
                                  : (const void *)d3::decode_select_fused_kernel<d3::kMaxK>;
    static int max_blocks[2] = {-1, -1};
    int &mb = max_blocks[n_extra <= 4 ? 0 : 1];
    if (mb < 0) {
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, d3::kThreads, smem);
        int dev = 0, sms = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        mb = per_sm * sms;
    }
    KVS_REQUIRE(mb > 0, KVS_ECUDA, "decode select kernel cannot be resident");
    int grid = mb < kNumSMs ? mb : kNumSMs;
    void *args[] = {(void *)&map_kv, (void *)&map_q, (void *)&p};
    cudaError_t e = cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(d3::kThreads), args,
                                                (size_t)smem, s);
    if (e != cudaSuccess) return cuda_status(e, "kvs_dhd_decode_select");
    return KVS_OK;
}

}  // namespace kvs
