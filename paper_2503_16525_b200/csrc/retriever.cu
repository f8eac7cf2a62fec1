// R1/R2 - the KV Retriever on the GPU.
//
// Reference semantics (pkg/src/kvlab/_matchcore.pyx:37-84, pool.py:125-161),
// restated data-parallel (SURVEY.md findings 1-2, verified on the oracle):
//   a target position t is claimed by the lexicographically smallest
//   (recency rank, j, i) over hash-equal window pairs (candidate window j of
//   that entry, target window i) whose token-equality run from (i, j) covers
//   t; its cached row is j + t - i.
// The kernel walks every target window i, probes the pool's sorted window
// hashes with a warp-wide 32-ary search, skips pairs dominated by their
// diagonal predecessor (i-1, j-1) (which covers a superset and is smaller),
// measures the run with ballots and claims positions with a 64-bit atomicMin
// on the packed key rank:22 | j:21 | i:21.
#include <cub/cub.cuh>

#include "common.cuh"

namespace kvs {

constexpr int kPosBits = 21;
constexpr uint64_t kPosMask = (1ull << kPosBits) - 1;
constexpr int64_t kMaxPos = (int64_t)1 << kPosBits;
constexpr int32_t kMaxRank = 1 << 22;
constexpr uint64_t kNoClaim = ~0ull;

__device__ __forceinline__ uint64_t mulmod(uint64_t a, uint64_t b, uint64_t m, bool small) {
    if (small) return (a * b) % m;  // a, b < 2^31
    return (uint64_t)(((unsigned __int128)a * b) % m);
}

// Windows [c*C, c*C + C) of request r: first hashed from scratch, then rolled
// (_matchcore.pyx:26-33).  blockIdx.y = request.
constexpr int kHashChunk = 32;
// off == nullptr: a single sequence of n_single tokens.
__global__ void window_hash_kernel(const int64_t *__restrict__ tok, const int64_t *__restrict__ off,
                                   int64_t n_single, int32_t w, uint64_t b, uint64_t m, uint64_t bw,
                                   uint64_t *__restrict__ out) {
    const int r = blockIdx.y;
    const int64_t s = off ? off[r] : 0, n = off ? off[r + 1] - off[r] : n_single;
    const int64_t nwin = n - w + 1;
    if (nwin <= 0) return;
    const bool small = m < (1ull << 31);
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c * kHashChunk < nwin;
         c += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i0 = c * kHashChunk;
        const int64_t i1 = min(nwin, i0 + kHashChunk);
        uint64_t h = 0;
        for (int k = 0; k < w; ++k)
            h = (mulmod(h, b, m, small) + ((uint64_t)tok[s + i0 + k]) % m) % m;
        out[s + i0] = h;  // indexed by the flat position of the window start
        for (int64_t i = i0 + 1; i < i1; ++i) {
            uint64_t drop = mulmod(((uint64_t)tok[s + i - 1]) % m, bw, m, small);
            h = (mulmod((h + m - drop) % m, b, m, small) + ((uint64_t)tok[s + i + w - 1]) % m) % m;
            out[s + i] = h;
        }
    }
}

static uint64_t host_powmod(uint64_t b, int64_t e, uint64_t m) {
    unsigned __int128 r = 1 % m, x = b % m;
    while (e > 0) {
        if (e & 1) r = (r * x) % m;
        x = (x * x) % m;
        e >>= 1;
    }
    return (uint64_t)r;
}

// Warp-cooperative lower_bound over a sorted u64 array (32-ary search).
__device__ __forceinline__ int64_t warp_lower_bound(const uint64_t *__restrict__ a, int64_t n,
                                                    uint64_t key) {
    const int lane = threadIdx.x & 31;
    int64_t lo = 0, hi = n;  // answer in [lo, hi]
    while (hi - lo > 32) {
        const int64_t step = (hi - lo + 31) / 32;
        const int64_t p = lo + (int64_t)lane * step;
        const bool less = (p < hi) && (a[p] < key);
        const uint32_t bal = __ballot_sync(0xffffffffu, less);
        // lanes [0, cnt) probe positions < key (monotone)
        const int cnt = __popc(bal);
        const int64_t nlo = cnt == 0 ? lo : lo + (int64_t)(cnt - 1) * step + 1;
        const int64_t nhi = cnt == 32 ? hi : min(hi, lo + (int64_t)cnt * step);
        lo = nlo;
        hi = nhi;
    }
    const int64_t p = lo + lane;
    const bool less = (p < hi) && (a[p] < key);
    return lo + __popc(__ballot_sync(0xffffffffu, less));
}

// One warp per target window (flat position t = start of window i of request r).
__global__ void __launch_bounds__(256) claim_kernel(
    kvs_token_index idx, const int64_t *__restrict__ req_tok, const int64_t *__restrict__ req_off,
    int32_t n_req, int64_t n_total, const uint64_t *__restrict__ th,
    unsigned long long *__restrict__ best) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int32_t w = idx.w;
    for (int64_t t = warp; t < n_total; t += nwarps) {
        // request of t (binary search over req_off, lane-uniform)
        int lo = 0, hi = n_req;  // req_off[lo] <= t < req_off[hi]
        while (hi - lo > 1) {
            int mid = (lo + hi) >> 1;
            if (req_off[mid] <= t) lo = mid; else hi = mid;
        }
        const int64_t s = req_off[lo], n_r = req_off[lo + 1] - s, i = t - s;
        if (i + w > n_r) continue;
        const uint64_t h = th[t];
        const int64_t b0 = warp_lower_bound(idx.sorted_hash, idx.n_windows, h);
        for (int64_t p = b0; p < idx.n_windows; ++p) {
            if (idx.sorted_hash[p] != h) break;
            const int32_t widx = idx.sorted_widx[p];
            const int32_t e = idx.win_slot[widx];
            const int32_t rank = idx.slot_rank[e];
            if (rank < 0) continue;
            const int64_t j = widx - idx.win_off[e];
            const int64_t es = idx.tok_off[e], n_e = idx.tok_off[e + 1] - es;
            // dominated by the diagonal predecessor pair (i-1, j-1)?
            if (i > 0 && j > 0 && req_tok[t - 1] == idx.tokens[es + j - 1] &&
                th[t - 1] == idx.win_hash[widx - 1])
                continue;
            const int64_t max_len = min(n_r - i, n_e - j);
            int64_t run = 0;
            for (int64_t base = 0; base < max_len; base += 32) {
                const int64_t k = base + lane;
                const bool eq = k < max_len && req_tok[t + k] == idx.tokens[es + j + k];
                const uint32_t bal = __ballot_sync(0xffffffffu, eq);
                if (bal != 0xffffffffu) {
                    run = base + __ffs(~bal) - 1;
                    break;
                }
                run = base + 32;
            }
            run = min(run, max_len);
            const unsigned long long key =
                ((unsigned long long)rank << (2 * kPosBits)) | ((uint64_t)j << kPosBits) | (uint64_t)i;
            for (int64_t k = lane; k < run; k += 32) atomicMin(&best[t + k], key);
        }
    }
}

__global__ void lookup_finalize_kernel(const unsigned long long *__restrict__ best,
                                       const int64_t *__restrict__ req_off, int32_t n_req,
                                       int64_t n_total, const int32_t *__restrict__ rank2slot,
                                       int32_t n_slots, int32_t *__restrict__ src_slot,
                                       int32_t *__restrict__ src_cand, int32_t *__restrict__ n_hit,
                                       uint8_t *__restrict__ contributed) {
    const int r = blockIdx.y;
    const int64_t s = req_off[r], n = req_off[r + 1] - s;
    int local = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long b = best[s + i];
        if (b == kNoClaim) {
            src_slot[s + i] = -1;
            src_cand[s + i] = -1;
        } else {
            const int32_t rank = (int32_t)(b >> (2 * kPosBits));
            const int64_t j = (b >> kPosBits) & kPosMask, i0 = b & kPosMask;
            const int32_t slot = rank2slot[rank];
            src_slot[s + i] = slot;
            src_cand[s + i] = (int32_t)(j + i - i0);
            if (contributed) contributed[(int64_t)r * n_slots + slot] = 1;
            ++local;
        }
    }
    local = warp_sum(local);
    if ((threadIdx.x & 31) == 0 && local) atomicAdd(&n_hit[r], local);
}

// match_pairs emission key: (j, i, t) ascending == the reference's discovery
// order (candidate windows j outer, bucket positions i inner, run offset k).
__global__ void emit_key_kernel(const unsigned long long *__restrict__ best, int64_t nt,
                                unsigned long long *__restrict__ keys) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nt;
         t += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long b = best[t];
        if (b == kNoClaim) {
            keys[t] = kNoClaim;
        } else {
            const uint64_t j = (b >> kPosBits) & kPosMask, i = b & kPosMask;
            keys[t] = (j << (2 * kPosBits)) | (i << kPosBits) | (uint64_t)t;
        }
    }
}

__global__ void emit_pairs_kernel(const unsigned long long *__restrict__ keys, int64_t nt,
                                  int64_t *__restrict__ tm, int64_t *__restrict__ cm,
                                  unsigned long long *__restrict__ count) {
    int local = 0;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nt;
         p += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long k = keys[p];
        if (k == kNoClaim) continue;
        const int64_t t = k & kPosMask, i = (k >> kPosBits) & kPosMask, j = k >> (2 * kPosBits);
        tm[p] = t;
        cm[p] = j + t - i;
        ++local;
    }
    local = warp_sum(local);
    if ((threadIdx.x & 31) == 0 && local) atomicAdd(count, (unsigned long long)local);
}

__global__ void iota_kernel(int32_t *a, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        a[i] = (int32_t)i;
}

__global__ void fill_u64_kernel(unsigned long long *a, int64_t n, unsigned long long v) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        a[i] = v;
}

__global__ void single_seq_index_kernel(int64_t nt, int64_t nc, int32_t w, int64_t *req_off,
                                        int64_t *tok_off, int64_t *win_off, int32_t *slot_rank,
                                        int32_t *rank2slot) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        req_off[0] = 0;
        req_off[1] = nt;
        tok_off[0] = 0;
        tok_off[1] = nc;
        win_off[0] = 0;
        win_off[1] = nc >= w ? nc - w + 1 : 0;
        slot_rank[0] = 0;
        rank2slot[0] = 0;
    }
}

static inline int grid_for(int64_t n, int threads, int max_blocks = kNumSMs * 16) {
    int64_t g = (n + threads - 1) / threads;
    if (g < 1) g = 1;
    if (g > max_blocks) g = max_blocks;
    return (int)g;
}

static inline size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

static size_t sort_pairs_bytes(int64_t n) {
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const uint64_t *)nullptr, (uint64_t *)nullptr,
                                    (const int32_t *)nullptr, (int32_t *)nullptr, (int)n);
    return bytes;
}
static size_t sort_keys_bytes(int64_t n) {
    size_t bytes = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, bytes, (const unsigned long long *)nullptr,
                                   (unsigned long long *)nullptr, (int)n);
    return bytes;
}

static kvs_status check_hash_params(int32_t w, uint64_t b, uint64_t m) {
    KVS_REQUIRE(w >= 1, KVS_EPARAM, "window_size must be >= 1, got %d", w);
    KVS_REQUIRE(b >= 2, KVS_EPARAM, "base must be >= 2");
    KVS_REQUIRE(m > b, KVS_EPARAM, "modulus must exceed base");
    KVS_REQUIRE(m < (1ull << 63), KVS_EPARAM, "modulus must be < 2^63");
    return KVS_OK;
}

}  // namespace kvs

using namespace kvs;

// F5 fixed-chunk baseline (reference pool.py:139-159 with fixed_chunk ->
// matching.py:171-194): target chunk i (positions [i*c, (i+1)*c), trailing
// partial chunk never matches) is claimed by the newest entry holding the
// identical block at a chunk-aligned offset, at the first such offset.  One
// warp per (request, chunk): entries in recency order, aligned candidate
// chunks ascending, lanes compare the block 32 tokens at a time.
__global__ void __launch_bounds__(128) fixed_chunk_kernel(
    kvs_token_index idx, const int64_t *__restrict__ tok, const int64_t *__restrict__ req_off,
    int32_t c, int32_t *__restrict__ src_slot, int32_t *__restrict__ src_cand,
    int32_t *__restrict__ n_hit, uint8_t *__restrict__ contributed) {
    const int lane = threadIdx.x & 31;
    const int r = blockIdx.y;
    const int64_t chunk = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    const int64_t s0 = req_off[r], n = req_off[r + 1] - s0;
    if ((chunk + 1) * c > n) return;
    const int64_t *blk = tok + s0 + chunk * c;
    for (int rank = 0; rank < idx.n_slots; ++rank) {
        const int32_t slot = idx.rank2slot[rank];
        if (idx.slot_rank[slot] != rank) break;          // past the live entries
        const int64_t e0 = idx.tok_off[slot], ne = idx.tok_off[slot + 1] - e0;
        for (int64_t j = 0; j + c <= ne; j += c) {
            bool eq = true;
            for (int k0 = 0; k0 < c && eq; k0 += 32) {
                const int k = k0 + lane;
                const bool ok = k >= c || blk[k] == idx.tokens[e0 + j + k];
                eq = __all_sync(0xffffffffu, ok);
            }
            if (eq) {
                for (int k = lane; k < c; k += 32) {
                    src_slot[s0 + chunk * c + k] = slot;
                    src_cand[s0 + chunk * c + k] = (int32_t)(j + k);
                }
                if (lane == 0) {
                    atomicAdd(&n_hit[r], c);
                    if (contributed) contributed[(int64_t)r * idx.n_slots + slot] = 1;
                }
                return;
            }
        }
    }
}

extern "C" {

kvs_status kvs_window_hashes(const int64_t *tokens, int64_t n, int32_t w, uint64_t b, uint64_t m,
                             uint64_t *out, kvs_stream_t stream) {
    kvs_status st = check_hash_params(w, b, m);
    if (st != KVS_OK) return st;
    if (n < w) return KVS_OK;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t chunks = (n - w + 1 + kHashChunk - 1) / kHashChunk;
    window_hash_kernel<<<dim3(grid_for(chunks, 128), 1), 128, 0, s>>>(
        tokens, nullptr, n, w, b, m, host_powmod(b, w - 1, m), out);
    KVS_CHECK_LAUNCH("kvs_window_hashes");
    return KVS_OK;
}

size_t kvs_match_pairs_workspace(int64_t nt, int64_t nc) {
    const int64_t nmax = nt > nc ? nt : nc;
    size_t b = 0;
    b += align256(sizeof(uint64_t) * (nt + 1));          // target window hashes (flat)
    b += align256(sizeof(uint64_t) * (nc + 1));          // candidate window hashes
    b += align256(sizeof(uint64_t) * (nc + 1));          // sorted hashes
    b += align256(sizeof(int32_t) * (nc + 1) * 3);       // widx iota, sorted widx, win_slot
    b += align256(sizeof(unsigned long long) * (nt + 1) * 3);  // best, keys, sorted keys
    b += align256(sizeof(int64_t) * 8 + sizeof(int32_t) * 8);  // offsets, ranks
    const size_t sp = sort_pairs_bytes(nmax + 1), sk = sort_keys_bytes(nt + 1);
    b += align256(sp > sk ? sp : sk);
    return b;
}

kvs_status kvs_match_pairs(const int64_t *target, int64_t nt, const int64_t *candidate, int64_t nc,
                           int32_t w, uint64_t b, uint64_t m, int64_t *tm, int64_t *cm,
                           int64_t *n_out, void *ws, size_t ws_bytes, kvs_stream_t stream) {
    kvs_status st = check_hash_params(w, b, m);
    if (st != KVS_OK) return st;
    KVS_REQUIRE(nt < kMaxPos && nc < kMaxPos, KVS_EPARAM,
                "sequences longer than 2^21 tokens are not supported");
    KVS_REQUIRE(ws_bytes >= kvs_match_pairs_workspace(nt, nc), KVS_EPARAM, "workspace too small");
    cudaStream_t s = (cudaStream_t)stream;
    cudaMemsetAsync(n_out, 0, sizeof(int64_t), s);
    if (nt < w || nc < w) return KVS_OK;
    char *p = (char *)ws;
    auto take = [&](size_t bytes) { char *r = p; p += align256(bytes); return (void *)r; };
    uint64_t *th = (uint64_t *)take(sizeof(uint64_t) * (nt + 1));
    uint64_t *ch = (uint64_t *)take(sizeof(uint64_t) * (nc + 1));
    uint64_t *sh = (uint64_t *)take(sizeof(uint64_t) * (nc + 1));
    int32_t *ints = (int32_t *)take(sizeof(int32_t) * (nc + 1) * 3);
    int32_t *iota = ints, *swidx = ints + (nc + 1), *wslot = ints + 2 * (nc + 1);
    unsigned long long *best = (unsigned long long *)take(sizeof(unsigned long long) * (nt + 1) * 3);
    unsigned long long *keys = best + (nt + 1), *skeys = best + 2 * (nt + 1);
    char *meta = (char *)take(sizeof(int64_t) * 8 + sizeof(int32_t) * 8);
    int64_t *req_off = (int64_t *)meta;           // {0, nt}
    int64_t *tok_off = req_off + 2;               // {0, nc}
    int64_t *win_off = req_off + 4;               // {0, nc-w+1}
    int32_t *slot_rank = (int32_t *)(req_off + 8);
    int32_t *rank2slot = slot_rank + 1;
    size_t sort_bytes = ws_bytes - (size_t)(p - (char *)ws);
    void *sort_ws = p;

    single_seq_index_kernel<<<1, 32, 0, s>>>(nt, nc, w, req_off, tok_off, win_off, slot_rank,
                                             rank2slot);
    const uint64_t bw = host_powmod(b, w - 1, m);
    window_hash_kernel<<<dim3(grid_for((nt - w + 1 + kHashChunk - 1) / kHashChunk, 128), 1), 128, 0, s>>>(
        target, nullptr, nt, w, b, m, bw, th);
    window_hash_kernel<<<dim3(grid_for((nc - w + 1 + kHashChunk - 1) / kHashChunk, 128), 1), 128, 0, s>>>(
        candidate, nullptr, nc, w, b, m, bw, ch);
    const int64_t ncw = nc - w + 1;
    iota_kernel<<<grid_for(ncw, 256), 256, 0, s>>>(iota, ncw);
    cudaMemsetAsync(wslot, 0, sizeof(int32_t) * ncw, s);
    if (cub::DeviceRadixSort::SortPairs(sort_ws, sort_bytes, ch, sh, iota, swidx, (int)ncw, 0, 64,
                                        s) != cudaSuccess)
        return cuda_status(cudaGetLastError(), "kvs_match_pairs sort");
    fill_u64_kernel<<<grid_for(nt, 256), 256, 0, s>>>(best, nt, kNoClaim);
    kvs_token_index idx;
    idx.n_slots = 1;
    idx.n_windows = ncw;
    idx.w = w;
    idx.b = b;
    idx.m = m;
    idx.tokens = candidate;
    idx.tok_off = tok_off;
    idx.win_off = win_off;
    idx.win_hash = ch;
    idx.win_slot = wslot;
    idx.sorted_hash = sh;
    idx.sorted_widx = swidx;
    idx.slot_rank = slot_rank;
    idx.rank2slot = rank2slot;
    claim_kernel<<<grid_for(nt * 32, 256, kNumSMs * 8), 256, 0, s>>>(idx, target, req_off, 1, nt, th,
                                                                       best);
    emit_key_kernel<<<grid_for(nt, 256), 256, 0, s>>>(best, nt, keys);
    if (cub::DeviceRadixSort::SortKeys(sort_ws, sort_bytes, keys, skeys, (int)nt, 0, 64, s) !=
        cudaSuccess)
        return cuda_status(cudaGetLastError(), "kvs_match_pairs emit sort");
    emit_pairs_kernel<<<grid_for(nt, 256), 256, 0, s>>>(skeys, nt, tm, cm,
                                                         (unsigned long long *)n_out);
    KVS_CHECK_LAUNCH("kvs_match_pairs");
    return KVS_OK;
}

size_t kvs_index_sort_workspace(int64_t n_windows) {
    return align256(sizeof(int32_t) * (n_windows + 1)) + align256(sort_pairs_bytes(n_windows + 1));
}

kvs_status kvs_index_sort(const uint64_t *win_hash, int64_t n_windows, uint64_t *sorted_hash,
                          int32_t *sorted_widx, void *ws, size_t ws_bytes, kvs_stream_t stream) {
    KVS_REQUIRE(ws_bytes >= kvs_index_sort_workspace(n_windows), KVS_EPARAM, "workspace too small");
    if (n_windows <= 0) return KVS_OK;
    cudaStream_t s = (cudaStream_t)stream;
    int32_t *iota = (int32_t *)ws;
    void *sort_ws = (char *)ws + align256(sizeof(int32_t) * (n_windows + 1));
    size_t sort_bytes = ws_bytes - align256(sizeof(int32_t) * (n_windows + 1));
    iota_kernel<<<grid_for(n_windows, 256), 256, 0, s>>>(iota, n_windows);
    if (cub::DeviceRadixSort::SortPairs(sort_ws, sort_bytes, win_hash, sorted_hash, iota,
                                        sorted_widx, (int)n_windows, 0, 64, s) != cudaSuccess)
        return cuda_status(cudaGetLastError(), "kvs_index_sort");
    KVS_CHECK_LAUNCH("kvs_index_sort");
    return KVS_OK;
}

size_t kvs_pool_lookup_workspace(int64_t n_total) {
    return align256(sizeof(uint64_t) * (n_total + 1)) +
           align256(sizeof(unsigned long long) * (n_total + 1));
}

kvs_status kvs_pool_lookup(const kvs_token_index *index, const int64_t *req_tokens,
                           const int64_t *req_off, int32_t n_req, int64_t n_total,
                           int32_t *src_slot, int32_t *src_cand, int32_t *n_hit,
                           uint8_t *contributed, void *ws, size_t ws_bytes,
                           kvs_stream_t stream) {
    KVS_REQUIRE(index != nullptr, KVS_EPARAM, "null index");
    kvs_status st = check_hash_params(index->w, index->b, index->m);
    if (st != KVS_OK) return st;
    KVS_REQUIRE(n_req >= 1 && n_req <= 65535, KVS_EPARAM, "n_req must be in [1, 65535]");
    KVS_REQUIRE(index->n_slots < kMaxRank, KVS_EPARAM, "too many pool slots");
    KVS_REQUIRE(ws_bytes >= kvs_pool_lookup_workspace(n_total), KVS_EPARAM, "workspace too small");
    cudaStream_t s = (cudaStream_t)stream;
    cudaMemsetAsync(n_hit, 0, sizeof(int32_t) * n_req, s);
    if (contributed && index->n_slots > 0)
        cudaMemsetAsync(contributed, 0, (size_t)n_req * index->n_slots, s);
    if (n_total <= 0) return KVS_OK;
    uint64_t *th = (uint64_t *)ws;
    unsigned long long *best =
        (unsigned long long *)((char *)ws + align256(sizeof(uint64_t) * (n_total + 1)));
    fill_u64_kernel<<<grid_for(n_total, 256), 256, 0, s>>>(best, n_total, kNoClaim);
    if (index->n_windows > 0 && index->n_slots > 0) {
        const uint64_t bw = host_powmod(index->b, index->w - 1, index->m);
        window_hash_kernel<<<dim3(4, n_req), 128, 0, s>>>(req_tokens, req_off, 0, index->w,
                                                           index->b, index->m, bw, th);
        claim_kernel<<<grid_for(n_total * 32, 256, kNumSMs * 8), 256, 0, s>>>(
            *index, req_tokens, req_off, n_req, n_total, th, best);
    }
    lookup_finalize_kernel<<<dim3(8, n_req), 256, 0, s>>>(best, req_off, n_req, n_total,
                                                          index->rank2slot, index->n_slots,
                                                          src_slot, src_cand, n_hit, contributed);
    KVS_CHECK_LAUNCH("kvs_pool_lookup");
    return KVS_OK;
}

kvs_status kvs_fixed_chunk_lookup(const kvs_token_index *index, const int64_t *req_tokens,
                                  const int64_t *req_off, int32_t n_req, int64_t max_len,
                                  int32_t chunk, int32_t *src_slot, int32_t *src_cand,
                                  int32_t *n_hit, uint8_t *contributed, int64_t n_total,
                                  kvs_stream_t stream) {
    KVS_REQUIRE(index != nullptr, KVS_EPARAM, "null index");
    KVS_REQUIRE(chunk >= 1, KVS_EPARAM, "chunk_size must be >= 1, got %d", chunk);
    KVS_REQUIRE(n_req >= 1 && n_req <= 65535, KVS_EPARAM, "n_req must be in [1, 65535]");
    cudaStream_t s = (cudaStream_t)stream;
    cudaMemsetAsync(n_hit, 0, sizeof(int32_t) * n_req, s);
    if (contributed && index->n_slots > 0)
        cudaMemsetAsync(contributed, 0, (size_t)n_req * index->n_slots, s);
    if (n_total <= 0) return KVS_OK;
    cudaMemsetAsync(src_slot, 0xFF, sizeof(int32_t) * n_total, s);     // -1: miss
    cudaMemsetAsync(src_cand, 0xFF, sizeof(int32_t) * n_total, s);
    const int64_t chunks = max_len / chunk;
    if (chunks > 0 && index->n_slots > 0) {
        fixed_chunk_kernel<<<dim3((unsigned)((chunks + 3) / 4), n_req), 128, 0, s>>>(
            *index, req_tokens, req_off, chunk, src_slot, src_cand, n_hit, contributed);
    }
    KVS_CHECK_LAUNCH("kvs_fixed_chunk_lookup");
    return KVS_OK;
}

}  // extern "C"
