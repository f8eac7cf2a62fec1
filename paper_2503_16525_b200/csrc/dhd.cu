// D2 DHD-select, D3 decode-stage DHD and the SIMT few-row (decode) attention.
//
// D2 follows v_impact_scores' dv-L1 half and _take_top
//   (reference deviation.py:111-115, selection.py:51-77): HBM-bound pass over
//   the probe-layer V rows (cached vs fresh) of every reused position, then a
//   per-request radix select of the budget smallest 64-bit keys
//   (~score_bits << 32 | pos), i.e. score descending, position ascending.
// D3 follows select_decode_step (selection.py:80-105): unmasked softmax of
//   q_t . K over the whole current context per query head, mean over heads,
//   times the prefill dv-L1, top n_extra over the eligible rows.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace kvs {

struct ArenaC {
    const __nv_bfloat16 *base;
    int32_t L, G, D, P;
    __device__ __forceinline__ const __nv_bfloat16 *row(int64_t page, int layer, int kv,
                                                        int r) const {
        return base + ((((size_t)page * L + layer) * 2 + kv) * P + r) * (size_t)(G * D);
    }
};
static inline ArenaC arena_c(const kvs_kv_arena *a) {
    return ArenaC{(const __nv_bfloat16 *)a->base, a->num_layers, a->kv_heads, a->head_dim,
                  a->page_size};
}

__device__ __forceinline__ int find_req(const int64_t *req_off, int n_req, int64_t t) {
    int lo = 0, hi = n_req;
    while (hi - lo > 1) {
        int mid = (lo + hi) >> 1;
        if (req_off[mid] <= t) lo = mid; else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ float l1_diff8(const uint4 &a, const uint4 &b) {
    const __nv_bfloat162 *x = reinterpret_cast<const __nv_bfloat162 *>(&a);
    const __nv_bfloat162 *y = reinterpret_cast<const __nv_bfloat162 *>(&b);
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        float2 fx = __bfloat1622float2(x[k]), fy = __bfloat1622float2(y[k]);
        s += fabsf(fx.x - fy.x) + fabsf(fx.y - fy.y);
    }
    return s;
}

// ---------------------------------------------------------------- D2 pass 1
// One warp per flat position (grid-stride); 16-byte loads, 4 in flight/lane.
__global__ void __launch_bounds__(256) dv_score_kernel(
    const __nv_bfloat16 *__restrict__ v_true, const float *__restrict__ alpha,
    const int32_t *__restrict__ src_slot, int32_t layer, ArenaC A,
    const int64_t *__restrict__ req_off, int32_t n_req, int64_t n_total,
    const int32_t *__restrict__ block_table, int32_t max_pages, float *__restrict__ dv_l1,
    float *__restrict__ score) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int nvec = A.G * A.D / 8;
    for (int64_t t = warp; t < n_total; t += nwarps) {
        if (src_slot[t] < 0) {
            if (lane == 0) { dv_l1[t] = 0.f; score[t] = 0.f; }
            continue;
        }
        const int r = find_req(req_off, n_req, t);
        const int32_t pos = (int32_t)(t - req_off[r]);
        const int64_t page = block_table[(int64_t)r * max_pages + pos / A.P];
        const uint4 *vc = reinterpret_cast<const uint4 *>(A.row(page, layer, 1, pos % A.P));
        const uint4 *vt = reinterpret_cast<const uint4 *>(v_true + t * (int64_t)(A.G * A.D));
        float s = 0.f;
        for (int v0 = 0; v0 < nvec; v0 += 128) {
            uint4 a[4], b[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int v = v0 + k * 32 + lane;
                if (v < nvec) { a[k] = __ldg(vc + v); b[k] = __ldg(vt + v); }
            }
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (v0 + k * 32 + lane < nvec) s += l1_diff8(a[k], b[k]);
        }
        s = warp_sum(s);
        if (lane == 0) {
            dv_l1[t] = s;
            score[t] = alpha[t] * s;
        }
    }
}

// ---------------------------------------------------------------- D2 pass 2
// Per request radix select of the `budget` smallest keys.  One CTA / request.
__device__ __forceinline__ uint64_t sel_key(const float *score, const int32_t *src_slot,
                                            int64_t s, int64_t i) {
    if (src_slot[s + i] < 0) return ~0ull;
    const uint32_t bits = __float_as_uint(fmaxf(score[s + i], 0.f));
    return ((uint64_t)(~bits) << 32) | (uint64_t)i;
}

__global__ void __launch_bounds__(1024) radix_select_kernel(
    const float *__restrict__ score, const int32_t *__restrict__ src_slot,
    const int64_t *__restrict__ req_off, const int32_t *__restrict__ budget,
    uint8_t *__restrict__ selected) {
    __shared__ uint32_t hist[256];
    __shared__ uint64_t s_prefix;
    __shared__ int32_t s_k;
    const int r = blockIdx.x;
    const int64_t s = req_off[r], n = req_off[r + 1] - s;
    const int32_t B = budget[r];
    if (threadIdx.x == 0) { s_prefix = 0; s_k = B; }
    // prefix/mask of the key bits fixed so far (most significant first)
    uint64_t mask = 0;
    for (int pass = 0; pass < 8 && B > 0; ++pass) {
        const int shift = 56 - 8 * pass;
        for (int b = threadIdx.x; b < 256; b += blockDim.x) hist[b] = 0;
        __syncthreads();
        const uint64_t prefix = s_prefix;
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
            const uint64_t key = sel_key(score, src_slot, s, i);
            if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 0xff], 1u);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            int32_t k = s_k;
            uint32_t cum = 0;
            int digit = 0;
            for (; digit < 256; ++digit) {
                if (cum + hist[digit] >= (uint32_t)k) break;
                cum += hist[digit];
            }
            if (digit > 255) digit = 255;
            s_k = k - (int32_t)cum;
            s_prefix = prefix | ((uint64_t)digit << shift);
        }
        mask |= 0xffull << shift;
        __syncthreads();
    }
    const uint64_t thr = s_prefix;  // the B-th smallest key (keys are unique)
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const uint64_t key = sel_key(score, src_slot, s, i);
        selected[s + i] = (B > 0 && key != ~0ull && key <= thr) ? 1 : 0;
    }
}

// ---------------------------------------------------------------- D2 fused
// One persistent launch: CTAs pull 16-row stages (request-major) from an
// atomic work counter and stream dv-L1 x alpha for them (16 threads per row,
// 16-byte loads, all of a stage's loads in flight at once).  A per-request completion counter elects the CTA that
// finished a request's last chunk to run that request's top-B selection while
// the other CTAs keep streaming later requests.  Selection: 4 radix passes
// (8-bit digits) over the descending-score key ~bits(score) of the reused
// rows give the B-th score; rows strictly better are kept and the remaining
// budget is filled with the equal-score rows in ascending position order
// (selection.py:63-66 tie rule) by an ordered block scan.
constexpr int kSelThreads = 256;

constexpr int kSelSmemKeys = 16384;   // requests up to 16k tokens select from smem

// Descending-score key; non-reused rows get the largest key.  (Scores are
// finite and >= 0; a denormal score ties with 0 - below any bf16 signal.)
__device__ __forceinline__ uint32_t sel_key32(const float *score, const int32_t *src_slot,
                                              int64_t t) {
    if (__ldcg(src_slot + t) < 0) return 0xFFFFFFFFu;
    const uint32_t k = ~__float_as_uint(fmaxf(__ldcg(score + t), 0.f));   // written by other CTAs
    return k < 0xFFFFFFFEu ? k : 0xFFFFFFFEu;
}

template <bool kSmem>
__device__ __noinline__ void select_request(const float *__restrict__ score, const int32_t *__restrict__ src_slot,
                               int64_t s, int64_t n, int32_t B, uint8_t *__restrict__ selected,
                               uint32_t *keys, uint32_t *hist, uint32_t *sh) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    constexpr int NW = kSelThreads / 32;
    if (B <= 0) {
        for (int64_t i = tid; i < n; i += kSelThreads) selected[s + i] = 0;
        return;
    }
    if (kSmem) {
        // 8 independent loads of each array in flight per thread
        for (int64_t b0 = 0; b0 < n; b0 += 8 * kSelThreads) {
            int32_t sl[8];
            float sc[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int64_t i = b0 + u * kSelThreads + tid;
                sl[u] = i < n ? __ldcg(src_slot + s + i) : -1;
                sc[u] = i < n ? __ldcg(score + s + i) : 0.f;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int64_t i = b0 + u * kSelThreads + tid;
                if (i < n) {
                    const uint32_t k = ~__float_as_uint(fmaxf(sc[u], 0.f));
                    keys[i] = sl[u] < 0 ? 0xFFFFFFFFu : (k < 0xFFFFFFFEu ? k : 0xFFFFFFFEu);
                }
            }
        }
        __syncthreads();
    }
    auto key_at = [&](int64_t i) -> uint32_t {
        return kSmem ? keys[i] : sel_key32(score, src_slot, s + i);
    };
    if (tid == 0) { sh[0] = 0; sh[1] = (uint32_t)B; }
    __shared__ uint32_t wsum[NW];
    uint32_t mask = 0;
    // 4 radix passes (8-bit digits, most significant first) find the B-th
    // smallest key; histograms by plain shared atomics (same-bin lanes of a
    // warp serialise in the atomic unit, far cheaper than match.any)
    for (int pass = 0; pass < 4; ++pass) {
        const int shift = 24 - 8 * pass;
        hist[tid] = 0;
        __syncthreads();
        const uint32_t prefix = sh[0];
        const int64_t nr = (n + 31) & ~(int64_t)31;      // whole warps stay converged
        for (int64_t i = tid; i < nr; i += kSelThreads) {
            const uint32_t key = i < n ? key_at(i) : 0xFFFFFFFFu;
            const bool in = key != 0xFFFFFFFFu && (key & mask) == prefix;
            const uint32_t bin = (key >> shift) & 0xff;
            // scores cluster in a few digits (same exponent): the bin of the
            // first active lane is counted with one atomic per warp, the
            // rest individually
            const uint32_t act = __ballot_sync(0xffffffffu, in);
            if (act == 0) continue;
            const uint32_t lead = __shfl_sync(0xffffffffu, bin, __ffs(act) - 1);
            const uint32_t same = __ballot_sync(0xffffffffu, in && bin == lead);
            if (lane == __ffs(act) - 1) atomicAdd(&hist[lead], (uint32_t)__popc(same));
            if (in && bin != lead) atomicAdd(&hist[bin], 1u);
        }
        __syncthreads();
        const uint32_t c = hist[tid];
        uint32_t incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) wsum[wid] = incl;
        __syncthreads();
        uint32_t base = 0;
        for (int w = 0; w < wid; ++w) base += wsum[w];
        const uint32_t excl = base + incl - c;
        const uint32_t k = sh[1];
        __syncthreads();
        if (c > 0 && excl < k && excl + c >= k) {
            sh[0] = prefix | ((uint32_t)tid << shift);
            sh[1] = k - excl;
        }
        mask |= 0xffu << shift;
        __syncthreads();
    }
    const uint32_t thr = sh[0], ties_needed = sh[1];
    // ties at the threshold key are taken in ascending position order
    // (selection.py:63-66): warp w owns the contiguous range [a, b) and walks
    // it 32 keys at a time, so ballots give each tie its rank in order
    const int64_t per = (n + NW - 1) / NW;
    const int64_t a = wid * per, b = min(n, a + per);
    uint32_t mine = 0;
    for (int64_t i0 = a; i0 < b; i0 += 32) {
        const int64_t i = i0 + lane;
        mine += __popc(__ballot_sync(0xffffffffu, i < b && key_at(i) == thr));
    }
    if (lane == 0) wsum[wid] = mine;
    __syncthreads();
    uint32_t before = 0;
    for (int w = 0; w < wid; ++w) before += wsum[w];
    const uint32_t lt = (1u << lane) - 1u;
    for (int64_t i0 = a; i0 < b; i0 += 32) {
        const int64_t i = i0 + lane;
        const uint32_t key = i < b ? key_at(i) : 0xFFFFFFFFu;
        const uint32_t tie = __ballot_sync(0xffffffffu, i < b && key == thr);
        bool keep = key < thr;
        if (i < b && key == thr) keep = before + __popc(tie & lt) < ties_needed;
        before += __popc(tie);
        if (i < b) selected[s + i] = keep ? 1 : 0;
    }
}

// Diagnostic phase timeline (KVS_SEL_TRACE builds only): %globaltimer stamps
// per CTA, read back with kvs_sel_trace_dump().
#ifdef KVS_SEL_TRACE
__device__ unsigned long long g_sel_trace[1024 * 8];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define SEL_TRACE(ph) \
    do { if (threadIdx.x == 0 && blockIdx.x < 1024) g_sel_trace[blockIdx.x * 8 + (ph)] = gtimer(); } while (0)
#else
#define SEL_TRACE(ph) do {} while (0)
#endif

// Selection of one request's top-B (selection.py:63-77) by one CTA, keys in
// shared memory (position i at keys[i]).  Key = ~bits(score): ascending key
// = descending score; bit 31 is set for every reused row and non-reused rows
// are 0xFFFFFFFF.  Digits below bit 31: the 8 exponent bits, then 8 + 8 + 7
// mantissa bits.
//   pass 0  exponent digit, per-warp histograms (scores cluster in a few
//           exponents, so one aggregated atomic counts most of a warp)
//   then    the threshold exponent's rows are compacted to l1 (key, pos);
//           the next digit is counted there with ballots into per-lane
//           registers (no shared atomics on spread digits); the rows
//           sharing the resulting 17-bit prefix (within 2^-8 of the B-th
//           score; typically a handful) are ranked pairwise by (key, pos),
//           which is the reference's ascending-position tie rule
//   else    (many near-ties or no room) the remaining digits over all keys
//           and an ordered tie pass.
// The code is kept small on purpose: only the last CTAs of the fused launch
// run it, cold, and instruction fetch dominated an unrolled version.
// The fused launch's selectors run the shared-memory-key (rolled-loop) path
// even for requests that fit the register path: only 1-8 CTAs run it, once per
// step, with its code evicted by the step's other kernels, and inside a real
// step the unrolled register variant's cold instruction fetch cost twice its
// arithmetic (16 vs 8 us; tools/select_trace_step.py).
#ifndef KVS_SEL_REG
#define KVS_SEL_REG 0
#endif
constexpr int kPairCap = 256;     // threshold-digit rows ranked pairwise
constexpr int kKPT = 16;          // register keys per thread
constexpr int kRegKeys = kKPT * kSelThreads;

template <bool kReg>
__device__ __noinline__ void select_fast(const float *__restrict__ score,
                                         const int32_t *__restrict__ src_slot, int64_t s, int64_t n,
                                         int32_t B, uint8_t *__restrict__ selected,
                                         uint32_t *whist /* [8][256] */, uint32_t *keys /* n, smem */,
                                         uint32_t *sh, uint2 *l1 /* smem */, int l1_cap,
                                         const uint32_t *__restrict__ pkeys /* nullable */) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    constexpr int NW = kSelThreads / 32;
    __shared__ uint32_t wsum[NW];
    __shared__ uint2 cand[kPairCap];
    __shared__ uint32_t s_nc;
    // keys of positions tid + 256k: registers (kReg, n <= kRegKeys) or smem
    const int nk = kReg ? kKPT : (int)((n + kSelThreads - 1) / kSelThreads);
    uint32_t kr[kReg ? kKPT : 1];
#pragma unroll(kReg ? 1 : 1)
    for (int k0 = 0; k0 < nk; k0 += 16) {
        uint32_t v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            const int64_t i = tid + (int64_t)(k0 + u) * kSelThreads;
            if (pkeys != nullptr) {
                v[u] = i < n ? __ldcg(pkeys + s + i) : 0xFFFFFFFFu;
            } else {
                const int32_t sl = i < n ? __ldcg(src_slot + s + i) : -1;
                const float sc = i < n ? __ldcg(score + s + i) : 0.f;
                const uint32_t x = ~__float_as_uint(fmaxf(sc, 0.f));
                v[u] = sl < 0 ? 0xFFFFFFFFu : (x < 0xFFFFFFFEu ? x : 0xFFFFFFFEu);
            }
        }
        if constexpr (kReg) {
#pragma unroll
            for (int u = 0; u < 16; ++u) kr[u] = v[u];
        } else {
#pragma unroll
            for (int u = 0; u < 16; ++u)
                if (k0 + u < nk) keys[tid + (k0 + u) * kSelThreads] = v[u];
        }
    }
    if constexpr (!kReg) __syncthreads();
    SEL_TRACE(5);
#define KEY(k) (kReg ? kr[(k) < kKPT ? (k) : 0] : ((k) < nk ? keys[tid + (k) * kSelThreads] : 0xFFFFFFFFu))
    if (B <= 0) {
        for (int64_t i = tid; i < n; i += kSelThreads) selected[s + i] = 0;
        return;
    }
    uint32_t prefix = 0x80000000u, mask = 0x80000000u, need = (uint32_t)B;
    uint32_t *wh = whist + wid * 256;
    bool compact = false;
    int n1 = 0;
#pragma unroll 1
    for (int pass = 0; pass < 4; ++pass) {
        const int shift = pass == 0 ? 23 : pass == 1 ? 15 : pass == 2 ? 7 : 0;
        const uint32_t dmask = pass == 3 ? 0x7fu : 0xffu;
        if (compact) {
            // lane L counts digits 8L..8L+7 of the compacted rows from ballots
            uint32_t cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll 1
            for (int a0 = wid * 32; a0 < n1; a0 += kSelThreads) {
                const int a = a0 + lane;
                const uint32_t d = a < n1 ? (l1[a].x >> shift) & dmask : 0u;
                const uint32_t inb = __ballot_sync(0xffffffffu, a < n1);
                uint32_t bb[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) bb[q] = __ballot_sync(0xffffffffu, (d >> q) & 1u);
                uint32_t hi = inb;
#pragma unroll
                for (int q = 3; q < 8; ++q) hi &= ((lane >> (q - 3)) & 1) ? bb[q] : ~bb[q];
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    cnt[q] += __popc(hi & ((q & 1) ? bb[0] : ~bb[0]) & ((q & 2) ? bb[1] : ~bb[1]) &
                                     ((q & 4) ? bb[2] : ~bb[2]));
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) wh[lane * 8 + q] = cnt[q];
        } else {
#pragma unroll
            for (int w = 0; w < NW; ++w) whist[w * 256 + tid] = 0;
            __syncthreads();
            // four keys per step: independent ballot/shuffle chains overlap
#pragma unroll(kReg ? kKPT / 4 : 1)
            for (int k0 = 0; k0 < nk; k0 += 4) {
                uint32_t bin[4], lead[4], same[4];
                bool in[4];
                int first[4];
#pragma unroll
                for (int g = 0; g < 4; ++g) {
                    const uint32_t key = KEY(k0 + g);
                    in[g] = key != 0xFFFFFFFFu && (key & mask) == prefix;
                    bin[g] = (key >> shift) & dmask;
                }
#pragma unroll
                for (int g = 0; g < 4; ++g) first[g] = __ffs(__ballot_sync(0xffffffffu, in[g])) - 1;
#pragma unroll
                for (int g = 0; g < 4; ++g) lead[g] = __shfl_sync(0xffffffffu, bin[g], first[g] & 31);
#pragma unroll
                for (int g = 0; g < 4; ++g)
                    same[g] = __ballot_sync(0xffffffffu, in[g] && bin[g] == lead[g]);
#pragma unroll
                for (int g = 0; g < 4; ++g) {
                    if (lane == first[g]) atomicAdd(&wh[lead[g]], (uint32_t)__popc(same[g]));
                    if (in[g] && bin[g] != lead[g]) atomicAdd(&wh[bin[g]], 1u);
                }
            }
        }
        __syncthreads();
        // prefix sum over the warp histograms: the digit holding the need-th
        // best key extends the prefix
        uint32_t c = 0;
#pragma unroll
        for (int w = 0; w < NW; ++w) c += whist[w * 256 + tid];
        uint32_t incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) wsum[wid] = incl;
        if (tid == 0) s_nc = 0;
        __syncthreads();
        uint32_t base = 0;
#pragma unroll
        for (int w = 0; w < NW; ++w) base += w < wid ? wsum[w] : 0u;
        const uint32_t excl = base + incl - c;
        if (c > 0 && excl < need && excl + c >= need) {
            sh[0] = prefix | ((uint32_t)tid << shift);
            sh[1] = need - excl;
            sh[2] = c;
        }
        __syncthreads();
        prefix = sh[0];
        need = sh[1];
        mask |= dmask << shift;
        const uint32_t cnt_t = sh[2];
        if (pass == 0) SEL_TRACE(7);
        if (pass == 0 && cnt_t <= (uint32_t)l1_cap) {
            // compact the threshold exponent's rows; decide all others now
#pragma unroll(kReg ? kKPT / 4 : 1)
            for (int k0 = 0; k0 < nk; k0 += 4) {
                uint32_t key[4], bal[4];
                bool in[4];
#pragma unroll
                for (int g = 0; g < 4; ++g) {
                    key[g] = KEY(k0 + g);
                    in[g] = key[g] != 0xFFFFFFFFu && (key[g] & mask) == prefix;
                    bal[g] = __ballot_sync(0xffffffffu, in[g]);
                }
                const uint32_t tot =
                    __popc(bal[0]) + __popc(bal[1]) + __popc(bal[2]) + __popc(bal[3]);
                uint32_t at = 0;
                if (lane == 0 && tot) at = atomicAdd(&s_nc, tot);
                at = __shfl_sync(0xffffffffu, at, 0);
                const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
                for (int g = 0; g < 4; ++g) {
                    const int64_t i = tid + (int64_t)(k0 + g) * kSelThreads;
                    if (in[g]) l1[at + __popc(bal[g] & lt)] = make_uint2(key[g], (uint32_t)i);
                    at += __popc(bal[g]);
                    if (!in[g] && i < n)
                        selected[s + i] = (key[g] != 0xFFFFFFFFu && key[g] < prefix) ? 1 : 0;
                }
            }
            __syncthreads();
            compact = true;
            n1 = (int)cnt_t;
        } else if (compact && cnt_t <= (uint32_t)kPairCap) {
            // rank the rows sharing the prefix pairwise; decide the rest of l1
#pragma unroll 1
            for (int a0 = wid * 32; a0 < n1; a0 += kSelThreads) {
                const int a = a0 + lane;
                const uint2 e = a < n1 ? l1[a] : make_uint2(0xFFFFFFFFu, 0u);
                const bool is_c = a < n1 && (e.x & mask) == prefix;
                const uint32_t bal = __ballot_sync(0xffffffffu, is_c);
                uint32_t at = 0;
                if (lane == 0 && bal) at = atomicAdd(&s_nc, (uint32_t)__popc(bal));
                at = __shfl_sync(0xffffffffu, at, 0) + __popc(bal & ((1u << lane) - 1u));
                if (is_c) cand[at] = e;
                else if (a < n1) selected[s + e.y] = (e.x & mask) < prefix ? 1 : 0;
            }
            __syncthreads();
            const int nc = (int)s_nc;
            for (int a = tid; a < nc; a += kSelThreads) {
                const uint2 me = cand[a];
                uint32_t rank = 0;
#pragma unroll 4
                for (int b = 0; b < nc; ++b) {
                    const uint2 o = cand[b];
                    rank += (o.x < me.x || (o.x == me.x && o.y < me.y)) ? 1u : 0u;
                }
                selected[s + me.y] = rank < need ? 1 : 0;
            }
            SEL_TRACE(6);
            return;
        } else {
            compact = false;       // many near-ties: finish over all keys
        }
    }
    const uint32_t thr = prefix;
    SEL_TRACE(6);
    // ties at the threshold: if every tie fits, no ordering is needed
    uint32_t mine = 0;
#pragma unroll(kReg ? kKPT : 1)
    for (int k = 0; k < nk; ++k) mine += KEY(k) == thr;
    uint32_t tot = mine;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
    if (lane == 0) wsum[wid] = tot;
    __syncthreads();
    uint32_t ties = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) ties += wsum[w];
    __syncthreads();
    if (ties == need) {
#pragma unroll(kReg ? kKPT : 1)
        for (int k = 0; k < nk; ++k) {
            const int64_t i = tid + (int64_t)k * kSelThreads;
            if (i < n) selected[s + i] = KEY(k) <= thr ? 1 : 0;
        }
        return;
    }
    // split tie band (selection.py:63-66, ascending position among equals):
    // position i = tid + 256k, so the order is k-major, then tid
#pragma unroll(kReg ? kKPT : 1)
    for (int k = 0; k < nk; ++k) {
        const uint32_t key = KEY(k);
        const bool tie = key == thr;
        const uint32_t bal = __ballot_sync(0xffffffffu, tie);
        if (lane == 0) wsum[wid] = __popc(bal);
        __syncthreads();
        uint32_t before = __popc(bal & ((1u << lane) - 1u)), total_k = 0;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            before += w < wid ? wsum[w] : 0u;
            total_k += wsum[w];
        }
        const int64_t i = tid + (int64_t)k * kSelThreads;
        if (i < n) selected[s + i] = (key < thr || (tie && before < need)) ? 1 : 0;
        need = need > total_k ? need - total_k : 0;
        __syncthreads();
    }
#undef KEY
}

// Streaming: stage = 16 rows of one request (16 | page size: one arena page).
// Thread t owns row t/16 and the 16-byte vectors v = t%16 + 16j of it in both
// V rows.  Stages are assigned round-robin (no atomics); each thread copies
// its own vectors with cp.async into a private slice of a kDepth-deep shared
// ring and consumes exactly those bytes, so the pipeline needs no barriers:
// stage k+kDepth-1's copies are in flight while stage k is reduced, and its
// metadata (liveness, page, alpha) was loaded one stage earlier still.
constexpr int kStageRows = 16;
constexpr int kVecPerThread = 8;          // 16 threads x 8 x 16 B = one 2 KB V row
constexpr int kDepth = 3;
constexpr size_t kStageBytes = (size_t)kSelThreads * kVecPerThread * 2 * 16;   // 64 KB
constexpr int kMetaQ = 1024;              // live-row queue entries (16 B each), power of 2
#ifndef KVS_CHUNK
#define KVS_CHUNK 128
#endif
constexpr int kChunkRows = KVS_CHUNK;     // rows per grabbed chunk (<= kSelThreads)
// requests up to kSmemKeys positions select with their keys in the (then idle) ring
constexpr int kSmemKeys = (int)((kDepth * kStageBytes - 8 * 1024) / 4) / kSelThreads * kSelThreads;

__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }


__global__ void __launch_bounds__(kSelThreads, 1) dhd_select_fused_kernel(
    const __nv_bfloat16 *__restrict__ v_true, const float *__restrict__ alpha,
    const int32_t *__restrict__ src_slot, int32_t layer, ArenaC A,
    const int64_t *__restrict__ req_off, int32_t n_req,
    const int32_t *__restrict__ budget, const int32_t *__restrict__ block_table,
    int32_t max_pages, float *__restrict__ dv_l1, float *__restrict__ score,
    uint8_t *__restrict__ selected, uint32_t *__restrict__ counters,
    uint32_t *__restrict__ keyws) {
    // counters[0] = CTAs that published their rows, counters[1] = selectors
    // done, counters[2] = chunks handed out (the last selector re-zeroes all); keyws[t] = the selection key of
    // row t (descending score, 0xFFFFFFFF for non-reused rows)
    extern __shared__ __align__(16) uint8_t s_ring[];            // kDepth x kStageBytes
    int64_t *ro = reinterpret_cast<int64_t *>(s_ring + kDepth * kStageBytes);   // n_req + 1
    __shared__ uint32_t sh[4];
    __shared__ int s_ticket;
    const int tid = threadIdx.x;
    SEL_TRACE(0);
    for (int r = tid; r <= n_req; r += kSelThreads) ro[r] = req_off[r];
    __syncthreads();
    const int64_t row_lo = ro[0], row_hi = ro[n_req];
    const int nvec = A.G * A.D / 8;           // 16-byte vectors per V row (<= 128)
    const int row = tid / 16, sub = tid % 16;
    // Work is handed out in chunks grabbed from a global counter, so CTAs
    // on SMs that see less bandwidth simply take fewer chunks.  Chunk c is
    // rows row_lo + c + NC*j (strided: reused spans are long, so contiguous
    // chunks would differ wildly in live rows); at most kSelThreads rows,
    // i.e. one row per thread.
    const int64_t n_rows = row_hi - row_lo;
    const int64_t nc_rows = (n_rows + kChunkRows - 1) / kChunkRows;
    const int64_t NC = nc_rows > 2 * (int64_t)gridDim.x ? nc_rows : 2 * (int64_t)gridDim.x;
    // Live rows of the grabbed chunks form one queue (mq, kMetaQ entries,
    // circular) that the copy ring streams through without draining between
    // chunks.  Chunk ids: blockIdx.x, then grid + blockIdx.x, then tickets
    // 2*grid + atomicAdd(counters[2]) fetched one chunk ahead, so neither
    // the ticket nor the next chunk's metadata loads stall the ring.
    struct RowMeta {
        int32_t t;        // flat row
        int32_t page;     // arena page of the cached row
        int32_t r;        // row in page
        float alpha;
    };
    RowMeta *mq = reinterpret_cast<RowMeta *>(ro + n_req + 1);
    // double-buffered by call parity: back-to-back calls must not reset the
    // values a slow thread of the previous call has yet to read
    __shared__ int s_live[2];
    __shared__ long long s_chunk[2];
    int par = 0;
    int64_t cur = blockIdx.x, nxt = (int64_t)gridDim.x + blockIdx.x;   // cur: loads in flight
    uint32_t ticket = 0;
    if (tid == 0) ticket = atomicAdd(&counters[2], 1u);
    bool p_live = false;
    int32_t p_page = 0, p_r = 0;
    float p_alpha = 0.f;
    int64_t p_t = -1;
    bool dep_done = false;
    auto issue_meta = [&](int64_t c) {
        p_t = -1;
        if (c >= NC || tid >= kChunkRows) return;
        const int64_t t = row_lo + c + NC * tid;
        if (t >= row_hi) return;
        int r = 0, hi = n_req;
        while (hi - r > 1) {
            const int mid = (r + hi) >> 1;
            if (ro[mid] <= t) r = mid; else hi = mid;
        }
        const int64_t i = t - ro[r];
        p_t = t;
        p_live = __ldg(src_slot + t) >= 0;
        p_page = __ldg(block_table + (int64_t)r * max_pages + i / A.P);
        if (!dep_done) {
            // launched as a programmatic dependent of D1's reduce: everything
            // above overlaps it; alpha is its output
            asm volatile("griddepcontrol.wait;" ::: "memory");
            dep_done = true;
        }
        p_alpha = __ldcg(alpha + t);
        p_r = (int32_t)(i % A.P);
    };
    // append chunk `cur`'s live rows to the queue, move on to the next chunk
    // (its loads go out now); returns the new tail
    auto finish_meta = [&](int tail) -> int {
        if (tid == 0) {
            s_live[par] = 0;
            s_chunk[par] = 2 * (long long)gridDim.x + ticket;
            ticket = atomicAdd(&counters[2], 1u);
        }
        __syncthreads();
        if (p_t >= 0) {
            if (p_live) {
                const int at = atomicAdd(&s_live[par], 1);
                mq[(tail + at) & (kMetaQ - 1)] = RowMeta{(int32_t)p_t, p_page, p_r, p_alpha};
            } else {
                dv_l1[p_t] = 0.f;
                score[p_t] = 0.f;
                keyws[p_t] = 0xFFFFFFFFu;
            }
        }
        __syncthreads();
        cur = nxt;
        nxt = s_chunk[par];
        issue_meta(cur);
        const int nt = tail + s_live[par];
        par ^= 1;
        return nt;
    };
    // ring layout [stage][j][array][thread][16 B]: a warp's accesses to one
    // (j, array) are 512 contiguous bytes (bank-conflict free)
    const uint32_t my_slice = smem_u32(s_ring) + tid * 16;
    auto issue = [&](int k, int slot, int tail) {
        const int e = k * kStageRows + row;
        if (e < tail) {
            const RowMeta m = mq[e & (kMetaQ - 1)];
            const uint4 *vc = reinterpret_cast<const uint4 *>(A.row(m.page, layer, 1, m.r));
            const uint4 *vt = reinterpret_cast<const uint4 *>(v_true + (int64_t)m.t * (A.G * A.D));
            const uint32_t dst = my_slice + (uint32_t)slot * (uint32_t)kStageBytes;
#pragma unroll
            for (int j = 0; j < kVecPerThread; ++j) {
                const int v = sub + 16 * j;
                if (v < nvec) {
                    cp_async16(dst + (2 * j) * (kSelThreads * 16), vc + v);
                    cp_async16(dst + (2 * j + 1) * (kSelThreads * 16), vt + v);
                }
            }
        }
        cp_async_commit();
    };

    int tail = 0;
    issue_meta(cur);
    if (!dep_done) {                 // threads without rows in the first chunk
        asm volatile("griddepcontrol.wait;" ::: "memory");
        dep_done = true;
    }
    tail = finish_meta(tail);
    SEL_TRACE(1);
    // keep the queue kDepth stages ahead of the stage being reduced
    auto refill = [&](int k_need) {
        while (tail < k_need * kStageRows && cur < NC) tail = finish_meta(tail);
    };
    refill(kDepth);
#pragma unroll
    for (int j = 0; j < kDepth - 1; ++j) issue(j, j, tail);
    for (int k0 = 0;; k0 += kDepth) {
        bool done = false;
#pragma unroll
        for (int u = 0; u < kDepth; ++u) {      // unrolled: ring slots are static
            const int k = k0 + u;
            if (k * kStageRows >= tail && cur >= NC) { done = true; break; }
            refill(k + kDepth);
            // copies for stage k+depth-1 go out before stage k is reduced
            issue(k + kDepth - 1, (u + kDepth - 1) % kDepth, tail);
            cp_async_wait<kDepth - 1>();
            const int e = k * kStageRows + row;
            float acc = 0.f;
            if (e < tail) {
                const uint8_t *src = s_ring + (size_t)u * kStageBytes + (size_t)tid * 16;
#pragma unroll
                for (int j = 0; j < kVecPerThread; ++j)
                    if (sub + 16 * j < nvec) {
                        const uint4 a =
                            *reinterpret_cast<const uint4 *>(src + (2 * j) * (kSelThreads * 16));
                        const uint4 b = *reinterpret_cast<const uint4 *>(
                            src + (2 * j + 1) * (kSelThreads * 16));
                        acc += l1_diff8(a, b);
                    }
            }
#pragma unroll
            for (int o = 8; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (e < tail && sub == 0) {
                const RowMeta m = mq[e & (kMetaQ - 1)];
                const float sc = m.alpha * acc;
                dv_l1[m.t] = acc;
                score[m.t] = sc;
                const uint32_t x = ~__float_as_uint(fmaxf(sc, 0.f));
                keyws[m.t] = x < 0xFFFFFFFEu ? x : 0xFFFFFFFEu;
            }
        }
        if (done) break;
    }
    cp_async_wait<0>();
    SEL_TRACE(2);
    // every CTA publishes its rows once; the last min(n_req, grid) CTAs to get
    // here become selectors, wait until all CTAs have published, and run one
    // request's top-B each (in parallel), so only one selection is exposed
    __threadfence();
    __syncthreads();
    if (tid == 0) s_ticket = (int)atomicAdd(&counters[0], 1u);
    __syncthreads();
    const int n_sel = n_req < (int)gridDim.x ? n_req : (int)gridDim.x;
    const int sel = s_ticket - ((int)gridDim.x - n_sel);
    if (sel < 0) return;
    if (tid == 0) {
        volatile uint32_t *done = counters;
        while (*done < gridDim.x) __nanosleep(32);
        __threadfence();
    }
    __syncthreads();
    SEL_TRACE(3);
    uint32_t *whist = reinterpret_cast<uint32_t *>(s_ring);           // the ring is free now
    uint32_t *keys = whist + kSelThreads / 32 * 256;
    for (int r = sel; r < n_req; r += n_sel) {
        const int64_t s0 = req_off[r], n = req_off[r + 1] - s0;
        constexpr int kFree = (int)(kDepth * kStageBytes / 4) - 8 * 256;   // words after whist
        if (KVS_SEL_REG && n <= kRegKeys) {
            select_fast<true>(score, src_slot, s0, n, budget[r], selected, whist, keys, sh,
                              reinterpret_cast<uint2 *>(keys), kFree / 2, keyws);
        } else if (n <= kSmemKeys) {
            const int nk2 = (int)((n + kSelThreads - 1) / kSelThreads * kSelThreads);   // keys[]
            select_fast<false>(score, src_slot, s0, n, budget[r], selected, whist, keys, sh,
                               reinterpret_cast<uint2 *>(keys + nk2), (kFree - nk2) / 2, keyws);
        }
        else
            select_request<false>(score, src_slot, s0, n, budget[r], selected, keys,
                                  keys + kSelSmemKeys, sh);
        __syncthreads();
    }
    SEL_TRACE(4);
    // the last selector out leaves the counters zeroed for the next launch
    if (tid == 0 && atomicAdd(&counters[1], 1u) + 1 == (uint32_t)n_sel) {
        counters[0] = 0;
        counters[1] = 0;
        counters[2] = 0;
        __threadfence();
    }
}

// F4: top-B over caller-given scores (reference selection.py:63-66 _take_top
// for the MAGNITUDE / RANDOM / IDEAL strategies, selection.py:154-183): one
// CTA per request; candidates are positions with cand >= 0, scores >= 0.
__global__ void __launch_bounds__(kSelThreads) topk_kernel(const float *__restrict__ score,
                                                           const int32_t *__restrict__ cand,
                                                           const int64_t *__restrict__ req_off,
                                                           const int32_t *__restrict__ budget,
                                                           uint8_t *__restrict__ selected,
                                                           int key_words, int l1_cap) {
    extern __shared__ uint32_t s_topk[];
    __shared__ uint32_t sh[4];
    const int r = blockIdx.x;
    const int64_t s = req_off[r], n = req_off[r + 1] - s;
    uint32_t *whist = s_topk, *keys = s_topk + 8 * 256;
    uint2 *l1 = reinterpret_cast<uint2 *>(keys + key_words);
    if (n <= kRegKeys)
        select_fast<true>(score, cand, s, n, budget[r], selected, whist, keys, sh, l1, l1_cap,
                          nullptr);
    else
        select_fast<false>(score, cand, s, n, budget[r], selected, whist, keys, sh, l1, l1_cap,
                           nullptr);
}

// ---------------------------------------------------------------- D3
// Pass 1: grid (request, key chunk).  Logits for all query heads of one key
// row, each K row read once for its GQA group; per-(request, chunk, head)
// partial max / sum-exp.
constexpr int kDecChunk = 256;    // keys per CTA of the logits pass (8 warps x 32)

// Pass 1: grid (key chunk, request, kv head), 8 warps, each a 32-key tile
// with one key per lane (a tile lies in one page).  The lane loads its key's
// 256-byte slice of the CTA's kv head and forms the HQ query heads' logits
// with q from shared memory; logits [request][head][key] (log2 domain) are
// written coalesced (consecutive keys per head).
template <int HQ>
__global__ void __launch_bounds__(256, 2) decode_logits_kernel(
    const __nv_bfloat16 *__restrict__ q_t, int32_t H, const int32_t *__restrict__ ctx_len,
    int32_t max_ctx, int32_t layer, ArenaC A, const int32_t *__restrict__ block_table,
    int32_t max_pages, float scale_log2, float *__restrict__ logits,
    float2 *__restrict__ part /* [request][tile][H] (max, sum) */) {
    constexpr int D = 128;
    __shared__ __align__(16) float sq[HQ * D];   // the group's query heads, fp32
    extern __shared__ __align__(16) uint8_t skey[];   // [warp][32 keys][256 B], swizzled
    // kv head fastest in the grid: the CTAs reading the 8 slices of the same
    // 2 KB key rows run together (DRAM row locality)
    const int g = blockIdx.x, r = blockIdx.z;
    const int n = ctx_len[r];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int t0 = blockIdx.y * kDecChunk + wid * 32;
    const int k = t0 + lane;
    const bool live = k < n;
    // The tile's 32 key slices (256 B each, 2 KB apart in the page) are
    // staged with cp.async so that every warp instruction moves two whole
    // slices (16 lanes x 16 B each) instead of 32 scattered 16-byte pieces;
    // chunk c of key j lands at slot c ^ (j & 15) (conflict-free reads of a
    // whole slice per lane below).  The K copies go out before q is staged.
    const uint32_t sk = smem_u32(skey) + wid * 8192;
    if (t0 < n) {
        const int64_t page = block_table[(int64_t)r * max_pages + t0 / A.P];
        const uint8_t *kbase =
            reinterpret_cast<const uint8_t *>(A.row(page, layer, 0, t0 % A.P) + g * D);
        const int c = lane & 15;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const int kk = 2 * j + (lane >> 4);
            if (t0 + kk < n)
                cp_async16(sk + kk * 256 + ((c ^ (kk & 15)) * 16),
                           kbase + (int64_t)kk * A.G * D * 2 + c * 16);
        }
        cp_async_commit();
    }
    for (int i = threadIdx.x; i < HQ * D; i += blockDim.x)
        sq[i] = bf2f(q_t[((int64_t)r * H + g * HQ) * D + i]);
    cp_async_wait<0>();
    __syncthreads();
    if (t0 >= n) return;
    uint4 kx[D / 8];
#pragma unroll
    for (int c = 0; c < D / 8; ++c) {
        const uint32_t addr = sk + lane * 256 + ((c ^ (lane & 15)) * 16);
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(kx[c].x), "=r"(kx[c].y), "=r"(kx[c].z), "=r"(kx[c].w)
                     : "r"(addr));
    }
    {
        float p[HQ];
#pragma unroll
        for (int hh = 0; hh < HQ; ++hh) p[hh] = 0.f;
#pragma unroll
        for (int c = 0; c < D / 8; ++c) {
            const __nv_bfloat162 *h2 = reinterpret_cast<const __nv_bfloat162 *>(&kx[c]);
            float kf[8];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const float2 f = __bfloat1622float2(h2[u]);
                kf[2 * u] = f.x;
                kf[2 * u + 1] = f.y;
            }
#pragma unroll
            for (int hh = 0; hh < HQ; ++hh) {
                const float *qh = sq + hh * D + 8 * c;
                const float4 qa = *reinterpret_cast<const float4 *>(qh);
                const float4 qb = *reinterpret_cast<const float4 *>(qh + 4);
                p[hh] += kf[0] * qa.x + kf[1] * qa.y + kf[2] * qa.z + kf[3] * qa.w +
                         kf[4] * qb.x + kf[5] * qb.y + kf[6] * qb.z + kf[7] * qb.w;
            }
        }
        const int tile = t0 / 32, n_tiles = (max_ctx + 31) / 32;
#pragma unroll
        for (int hh = 0; hh < HQ; ++hh) {
            const float x = live ? p[hh] * scale_log2 : -INFINITY;
            if (live) logits[((int64_t)r * H + g * HQ + hh) * ((max_ctx + 3) & ~3) + k] = x;
            const float mt = warp_max(x);
            const float z = warp_sum(live ? fast_exp2(x - mt) : 0.f);
            if (lane == 0) part[((int64_t)r * n_tiles + tile) * H + g * HQ + hh] = make_float2(mt, z);
        }
    }
}

// Pass 2: one CTA per request: per-head softmax statistics over the whole
// context (unmasked, selection.py:100-102) by block reductions, the mean
// head weight x dv-L1 of every prefill row into shared memory (decode rows
// have zero deviation, engine.py:145-147), then n_extra block-argmax rounds
// on (score desc, position asc) over the still-eligible rows.
__global__ void __launch_bounds__(1024) decode_select_kernel(
    int32_t H, const int32_t *__restrict__ ctx_len, int32_t max_ctx,
    const float *__restrict__ logits, const float2 *__restrict__ part,
    const float *__restrict__ dv_l1,
    uint8_t *__restrict__ eligible, const int64_t *__restrict__ req_off, int32_t n_extra,
    int32_t *__restrict__ chosen, int32_t *__restrict__ n_chosen, float *__restrict__ scores_out) {
    extern __shared__ float sc[];            // [max_ctx] scores of this request
    __shared__ float sm[64], sz[64];
    __shared__ uint64_t redk[32];
    __shared__ int32_t s_pick[64];
    const int r = blockIdx.x;
    const int n = ctx_len[r];
    const int64_t s = req_off[r];
    const int n_pre = (int)(req_off[r + 1] - s);
    {
        // warp w combines head w's per-tile (max, sum) partials of the logits pass
        const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
        const int n_tiles = (max_ctx + 31) / 32, used = (n + 31) / 32;
        for (int h = wid; h < H; h += blockDim.x >> 5) {
            float m = -INFINITY, z = 0.f;
            for (int t = lane; t < used; t += 32) {
                const float2 pz = part[((int64_t)r * n_tiles + t) * H + h];
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
            if (lane == 0) {
                sm[h] = m;
                sz[h] = 1.f / z;
            }
        }
    }
    __syncthreads();
    const float invH = 1.f / (float)H;
    float *scr = scores_out ? scores_out + (int64_t)r * max_ctx : nullptr;
    // four consecutive rows per thread: 16-byte loads of each head's logits
    // (L2-resident), eight heads in flight
    const int64_t ld = (max_ctx + 3) & ~3;
    for (int i0 = 4 * threadIdx.x; i0 < n; i0 += 4 * blockDim.x) {
        float w[4] = {0.f, 0.f, 0.f, 0.f};
        if (i0 < n_pre)
            for (int h0 = 0; h0 < H; h0 += 8) {
                float4 x[8];
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    x[u] = h0 + u < H ? __ldcg(reinterpret_cast<const float4 *>(
                                            logits + ((int64_t)r * H + h0 + u) * ld + i0))
                                      : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (h0 + u < H) {
                        const float mh = sm[h0 + u], zh = sz[h0 + u];
                        w[0] += fast_exp2(x[u].x - mh) * zh;
                        w[1] += fast_exp2(x[u].y - mh) * zh;
                        w[2] += fast_exp2(x[u].z - mh) * zh;
                        w[3] += fast_exp2(x[u].w - mh) * zh;
                    }
            }
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int i = i0 + e;
            if (i >= n) break;
            const float v = i < n_pre ? w[e] * invH * dv_l1[s + i] : 0.f;
            sc[i] = v;
            if (scr) scr[i] = v;
        }
    }
    __syncthreads();
    int picked = 0;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int round = 0; round < n_extra; ++round) {
        uint64_t best = ~0ull;
        for (int i = threadIdx.x; i < n_pre && i < n; i += blockDim.x) {
            if (!eligible[s + i]) continue;
            const uint64_t key = ((uint64_t)(~__float_as_uint(fmaxf(sc[i], 0.f))) << 32) | (uint32_t)i;
            best = key < best ? key : best;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const uint64_t x = __shfl_xor_sync(0xffffffffu, best, o);
            best = x < best ? x : best;
        }
        if (lane == 0) redk[wid] = best;
        __syncthreads();
        if (threadIdx.x == 0) {
            uint64_t b = ~0ull;
            for (int k = 0; k < (int)(blockDim.x >> 5); ++k) b = redk[k] < b ? redk[k] : b;
            s_pick[round] = b == ~0ull ? -1 : (int32_t)(b & 0xffffffffu);
            if (b != ~0ull) eligible[s + (b & 0xffffffffu)] = 0;
        }
        __syncthreads();
        if (s_pick[round] < 0) break;
        ++picked;
    }
    if (threadIdx.x == 0) {
        // ascending order (selection.py:66), pad with -1
        int32_t tmp[64];
        for (int k = 0; k < picked; ++k) tmp[k] = s_pick[k];
        for (int a = 1; a < picked; ++a)
            for (int b = a; b > 0 && tmp[b - 1] > tmp[b]; --b) {
                int32_t x = tmp[b]; tmp[b] = tmp[b - 1]; tmp[b - 1] = x;
            }
        for (int k = 0; k < n_extra; ++k)
            chosen[(int64_t)r * n_extra + k] = k < picked ? tmp[k] : -1;
        n_chosen[r] = picked;
    }
}

static inline size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }


}  // namespace kvs

using namespace kvs;

extern "C" int32_t kvs_sel_trace_dump(uint64_t *host, int32_t n) {
#ifdef KVS_SEL_TRACE
    const int m = n < 1024 * 8 ? n : 1024 * 8;
    cudaMemcpyFromSymbol(host, kvs::g_sel_trace, sizeof(uint64_t) * m);
    static unsigned long long zero[1024 * 8];
    cudaMemcpyToSymbol(kvs::g_sel_trace, zero, sizeof(zero));
    return m;
#else
    (void)host;
    (void)n;
    return -1;
#endif
}

extern "C" {

size_t kvs_dhd_select_workspace(int64_t n_total, int32_t n_req) {
    (void)n_req;
    // self-resetting counters, then one selection key per row
    return 256 + align256(sizeof(uint32_t) * (size_t)(n_total > 0 ? n_total : 0));
}

/* Workspace contract: the first 256 bytes of the workspace must be zero
 * before the first call on a buffer; the kernel leaves them zero again. */
kvs_status kvs_dhd_select(const void *v_true, const float *alpha, const int32_t *src_slot,
                          int32_t layer, const kvs_kv_arena *arena, const kvs_batch *batch,
                          const int32_t *budget, float *dv_l1, float *score, uint8_t *selected,
                          void *ws, size_t ws_bytes, kvs_stream_t stream) {
    KVS_REQUIRE(arena && batch, KVS_EPARAM, "null arena/batch");
    KVS_REQUIRE((arena->kv_heads * arena->head_dim) % 8 == 0, KVS_ESHAPE, "row width % 8 != 0");
    KVS_REQUIRE(ws != nullptr && ws_bytes >= kvs_dhd_select_workspace(batch->n_total, batch->n_req),
                KVS_EPARAM, "workspace too small (kvs_dhd_select_workspace)");
    if (batch->n_total <= 0) return KVS_OK;
    cudaStream_t s = (cudaStream_t)stream;
    uint32_t *counters = (uint32_t *)ws;
    // counters start zeroed (Workspace.get(zero=True)) and are re-zeroed by the kernel
    KVS_REQUIRE(arena->kv_heads * arena->head_dim <= 16 * kVecPerThread * 8, KVS_ESHAPE,
                "select: kv_heads * head_dim must be <= 1024");
    const size_t smem = kDepth * kStageBytes + sizeof(int64_t) * (batch->n_req + 1) +
                        16 * kMetaQ;
    KVS_REQUIRE(smem <= 227 * 1024, KVS_EPARAM, "select: too many requests in one batch");
    cudaFuncSetAttribute(dhd_select_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    // programmatic dependent launch: the prologue (request offsets, the first
    // chunk's liveness and page loads) overlaps the preceding kernel (D1's
    // reduce); the kernel waits for it before reading alpha
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(kNumSMs);
    lc.blockDim = dim3(kSelThreads);
    lc.dynamicSmemBytes = smem;
    lc.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = attr;
    lc.numAttrs = getenv("KVS_NO_PDL") == nullptr ? 1 : 0;
    cudaLaunchKernelEx(&lc, dhd_select_fused_kernel, (const __nv_bfloat16 *)v_true, alpha,
                       src_slot, layer, arena_c(arena), batch->req_off, batch->n_req, budget,
                       batch->block_table, batch->max_pages, dv_l1, score, selected, counters,
                       reinterpret_cast<uint32_t *>((uint8_t *)ws + 256));
    KVS_CHECK_LAUNCH("kvs_dhd_select");
    return KVS_OK;
}

size_t kvs_dhd_decode_select_workspace(int32_t n_req, int32_t num_heads, int32_t max_ctx) {
    const size_t tiles = ((size_t)max_ctx + 31) / 32;
    const size_t two_pass = kvs::d3_counter_bytes() +
        align256(sizeof(float) * (size_t)n_req * num_heads * (((size_t)max_ctx + 3) & ~(size_t)3)) +
        align256(sizeof(float2) * (size_t)n_req * tiles * num_heads);
    const size_t fused = kvs::d3_fused_workspace(n_req, num_heads, max_ctx);
    return two_pass > fused ? two_pass : fused;
}

kvs_status kvs_dhd_decode_select(const void *q_t, int32_t num_heads, const int32_t *ctx_len,
                                 int32_t max_ctx, const float *dv_l1, uint8_t *eligible,
                                 int32_t layer, const kvs_kv_arena *arena, const kvs_batch *batch,
                                 int32_t n_extra, float softmax_scale, int32_t *chosen,
                                 int32_t *n_chosen, float *scores, void *ws, size_t ws_bytes,
                                 kvs_stream_t stream) {
    KVS_REQUIRE(arena && batch, KVS_EPARAM, "null arena/batch");
    KVS_REQUIRE(num_heads <= 64 && num_heads % arena->kv_heads == 0, KVS_ESHAPE,
                "num_heads must be <= 64 and a multiple of kv_heads");
    KVS_REQUIRE(arena->head_dim == 128, KVS_ESHAPE, "head_dim must be 128 (padded heads)");
    KVS_REQUIRE(num_heads / arena->kv_heads <= 8, KVS_ESHAPE, "num_heads / kv_heads must be <= 8");
    KVS_REQUIRE(n_extra >= 0 && n_extra <= 64, KVS_EPARAM, "n_extra must be in [0, 64]");
    KVS_REQUIRE(ws_bytes >= kvs_dhd_decode_select_workspace(batch->n_req, num_heads, max_ctx),
                KVS_EPARAM, "workspace too small");
    cudaStream_t s = (cudaStream_t)stream;
    if (n_extra == 0 || max_ctx <= 0) {
        cudaMemsetAsync(n_chosen, 0, sizeof(int32_t) * batch->n_req, s);
        return KVS_OK;
    }
    if (kvs::d3_fused_supported(arena, batch->n_req, num_heads, n_extra))
        return kvs::d3_fused_launch(q_t, num_heads, ctx_len, max_ctx, dv_l1, eligible, layer, arena,
                                    batch, n_extra, softmax_scale, chosen, n_chosen, scores, ws, s);
    const int chunks = (max_ctx + kDecChunk - 1) / kDecChunk;
    // after the fused kernel's counter header, which stays zero
    float *logits = (float *)((char *)ws + kvs::d3_counter_bytes());
    float2 *part = (float2 *)((char *)logits + align256(sizeof(float) * (size_t)batch->n_req *
                                                     num_heads * (((size_t)max_ctx + 3) & ~(size_t)3)));
    const float scale_log2 = softmax_scale * 1.4426950408889634f;
    const int hq = num_heads / arena->kv_heads;
    const dim3 grid(arena->kv_heads, chunks, batch->n_req);     // one kv head per CTA
#define KVS_DECODE_LOGITS(HQ)                                                                  \
    cudaFuncSetAttribute(decode_logits_kernel<HQ>, cudaFuncAttributeMaxDynamicSharedMemorySize,  \
                         8 * 8192);                                                            \
    decode_logits_kernel<HQ><<<grid, 256, 8 * 8192, s>>>((const __nv_bfloat16 *)q_t, num_heads,    \
                                                     ctx_len, max_ctx, layer, arena_c(arena),  \
                                                     batch->block_table, batch->max_pages,     \
                                                     scale_log2, logits, part)
    switch (hq) {
        case 1: KVS_DECODE_LOGITS(1); break;
        case 2: KVS_DECODE_LOGITS(2); break;
        case 3: KVS_DECODE_LOGITS(3); break;
        case 4: KVS_DECODE_LOGITS(4); break;
        case 5: KVS_DECODE_LOGITS(5); break;
        case 6: KVS_DECODE_LOGITS(6); break;
        case 7: KVS_DECODE_LOGITS(7); break;
        default: KVS_DECODE_LOGITS(8); break;
    }
#undef KVS_DECODE_LOGITS
    const size_t sel_smem = sizeof(float) * (size_t)max_ctx;
    KVS_REQUIRE(sel_smem <= 200 * 1024, KVS_ESHAPE, "decode context longer than 51200 tokens");
    cudaFuncSetAttribute(decode_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sel_smem);
    decode_select_kernel<<<batch->n_req, 1024, sel_smem, s>>>(
        num_heads, ctx_len, max_ctx, logits, part, dv_l1, eligible, batch->req_off, n_extra,
        chosen, n_chosen, scores);
    KVS_CHECK_LAUNCH("kvs_dhd_decode_select");
    return KVS_OK;
}

kvs_status kvs_topk_select(const float *scores, const int32_t *cand, const int64_t *req_off,
                           int32_t n_req, int64_t max_len, const int32_t *budget,
                           uint8_t *selected, kvs_stream_t stream) {
    KVS_REQUIRE(n_req >= 1 && n_req <= 65535, KVS_EPARAM, "n_req must be in [1, 65535]");
    KVS_REQUIRE(max_len <= kSmemKeys, KVS_ESHAPE, "requests longer than %d positions", kSmemKeys);
    // keys[] holds whole rows of 256 (position tid + 256k)
    const int key_words = (int)((std::max<int64_t>(max_len, 1) + kSelThreads - 1) / kSelThreads *
                                kSelThreads);
    // compacted threshold-exponent rows: up to max_len entries while the
    // total stays within 200 KB (larger requests fall back to more passes)
    const int l1_cap = (int)std::min<int64_t>(
        std::max<int64_t>(max_len, 1), (200 * 1024 / 4 - 8 * 256 - key_words) / 2);
    const int smem = (int)(sizeof(uint32_t) * (8 * 256 + key_words + 2 * l1_cap));
    cudaFuncSetAttribute(topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    topk_kernel<<<n_req, kSelThreads, smem, (cudaStream_t)stream>>>(scores, cand, req_off, budget,
                                                                    selected, key_words, l1_cap);
    KVS_CHECK_LAUNCH("kvs_topk_select");
    return KVS_OK;
}

}  // extern "C"
