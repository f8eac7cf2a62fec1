/*
 * kvshare.h - C ABI of the B200-native KVShare DHD hot path (libkvshare.so).
 *
 * Plain pointers and sizes only: every buffer is caller-owned DEVICE memory
 * (the Python host passes torch tensor data pointers), every call is
 * asynchronous on the caller's stream, and hot calls never allocate (scratch
 * comes from a caller workspace sized by the matching *_workspace query).
 * Status codes map 1:1 onto the reference's error classes
 * (reference pkg/src/kvlab/errors.py:4-45); kvs_last_error() returns the
 * thread-local message of the last failure.
 *
 * Reference interfaces replaced (paths relative to reference pkg/src/kvlab):
 *   kvs_window_hashes     <- _matchcore.window_hashes   (_matchcore.pyx:16-34)
 *   kvs_match_pairs       <- _matchcore.match_pairs     (_matchcore.pyx:37-84)
 *   kvs_pool_lookup       <- CachePool.lookup           (pool.py:125-161)
 *   kvs_gather_kv         <- _forward / _perturbed_probe cached-row
 *                            substitution (model.py:196-200, engine.py:204-206)
 *   kvs_qkv_rope_scatter  <- split_heads(x @ W_{q,k,v}) (model.py:193-195)
 *                            + the KV write of _token_rows (engine.py:99-103)
 *   kvs_attention_fwd     <- attention_forward inside _forward on the query
 *                            rows it computes (model.py:110-129, 201)
 *   kvs_dhd_alpha         <- alpha of v_impact_scores   (deviation.py:108-110)
 *   kvs_dhd_select        <- dv-L1 x alpha + _take_top  (deviation.py:111-115,
 *                            selection.py:51-77)
 *   kvs_dhd_decode_select <- select_decode_step         (selection.py:80-105)
 *   kvs_decode_attention  <- the per-token attention of _token_rows /
 *                            query_rows_probe (engine.py:104-109, 164-168)
 */
#ifndef KVSHARE_H_
#define KVSHARE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *kvs_stream_t; /* == cudaStream_t */

typedef enum {
    KVS_OK = 0,
    KVS_EPARAM = 1,   /* kvlab.errors.ParameterError */
    KVS_ESHAPE = 2,   /* kvlab.errors.ShapeError     */
    KVS_EINPUT = 3,   /* kvlab.errors.InputError     */
    KVS_ECACHE = 4,   /* kvlab.errors.CacheError     */
    KVS_ENUMERIC = 5, /* kvlab.errors.NumericError   */
    KVS_ECUDA = 100   /* CUDA runtime / launch failure */
} kvs_status;

const char *kvs_last_error(void);
int32_t kvs_abi_version(void);

/* ------------------------------------------------------------------ R1/R2
 * Rolling-hash KV Retriever.  Tokens are int64 (non-negative; validated by
 * the host like matching.py:101-107).  Any prime modulus m > b is accepted
 * (64-bit residue products when m < 2^31, 128-bit otherwise).               */

/* out[i] = sum_k (tok[i+k] mod m) * b^(w-1-k) mod m, i < n-w+1 (0 outputs if n < w). */
kvs_status kvs_window_hashes(const int64_t *tokens, int64_t n, int32_t w, uint64_t b,
                             uint64_t m, uint64_t *out, kvs_stream_t stream);

/* Adaptive matcher, one target vs one candidate, reference claim order:
 * tm/cm hold <= nt pairs ordered exactly as _matchcore.match_pairs emits
 * them; *n_out (device int64) receives the count.                          */
size_t kvs_match_pairs_workspace(int64_t nt, int64_t nc);
kvs_status kvs_match_pairs(const int64_t *target, int64_t nt, const int64_t *candidate,
                           int64_t nc, int32_t w, uint64_t b, uint64_t m, int64_t *tm,
                           int64_t *cm, int64_t *n_out, void *ws, size_t ws_bytes,
                           kvs_stream_t stream);

/* Token-side index of the shared KV pool (replicated on every GPU).
 * Windows are numbered entry-major: window j of slot e is widx =
 * win_off[e] + j.  sorted_hash/sorted_widx list every live window by hash
 * (dead windows carry hash UINT64_MAX).  slot_rank[e] = recency rank
 * (0 = newest insert, pool.py:139), -1 for a free slot.                     */
typedef struct {
    int32_t n_slots;
    int64_t n_windows;
    int32_t w;
    uint64_t b, m;
    const int64_t *tokens;      /* concatenated entry tokens          */
    const int64_t *tok_off;     /* [n_slots+1]                        */
    const int64_t *win_off;     /* [n_slots+1]                        */
    const uint64_t *win_hash;   /* [n_windows] entry-major            */
    const int32_t *win_slot;    /* [n_windows]                        */
    const uint64_t *sorted_hash;/* [n_windows] ascending              */
    const int32_t *sorted_widx; /* [n_windows]                        */
    const int32_t *slot_rank;   /* [n_slots]                          */
    const int32_t *rank2slot;   /* [n_slots]                          */
} kvs_token_index;

size_t kvs_index_sort_workspace(int64_t n_windows);
kvs_status kvs_index_sort(const uint64_t *win_hash, int64_t n_windows, uint64_t *sorted_hash,
                          int32_t *sorted_widx, void *ws, size_t ws_bytes, kvs_stream_t stream);

/* Batched CachePool.lookup over n_req requests (flat tokens, req_off[n_req+1]).
 * Per flat position t: src_slot[t] (-1 = miss) and src_cand[t]; n_hit[r];
 * contributed[r * n_slots + e] = 1 when slot e claimed a position of r.    */
size_t kvs_pool_lookup_workspace(int64_t n_total);
kvs_status kvs_pool_lookup(const kvs_token_index *index, const int64_t *req_tokens,
                           const int64_t *req_off, int32_t n_req, int64_t n_total,
                           int32_t *src_slot, int32_t *src_cand, int32_t *n_hit,
                           uint8_t *contributed, void *ws, size_t ws_bytes,
                           kvs_stream_t stream);

/* ------------------------------------------------------------------ KV arena
 * One paged bf16 arena per GPU holds pool entries AND request caches:
 * page p, layer l, kv (0 = K, 1 = V), row r (< page_size), head g, dim i at
 * element ((((p * L + l) * 2 + kv) * page_size + r) * kv_heads + g) * head_dim + i.
 * K is stored post-RoPE at the owning sequence's positions.                */
/* F5 fixed-chunk baseline lookup (reference pool.py:125-161 with fixed_chunk,
 * matching.py:171-194): per request, chunk-aligned blocks of `chunk` tokens
 * (the trailing partial block never matches) claimed by the newest entry
 * holding the identical block at a chunk-aligned offset (first offset wins).
 * Same outputs as kvs_pool_lookup; max_len bounds the request lengths.     */
kvs_status kvs_fixed_chunk_lookup(const kvs_token_index *index, const int64_t *req_tokens,
                                  const int64_t *req_off, int32_t n_req, int64_t max_len,
                                  int32_t chunk, int32_t *src_slot, int32_t *src_cand,
                                  int32_t *n_hit, uint8_t *contributed, int64_t n_total,
                                  kvs_stream_t stream);

typedef struct {
    void *base;
    int64_t num_pages;
    int32_t num_layers, kv_heads, head_dim, page_size;
} kvs_kv_arena;

/* Flat batch of sequences: tokens t in [req_off[r], req_off[r+1]) belong to
 * request r; block_table[r * max_pages + k] = arena page of positions
 * [k*page_size, (k+1)*page_size).                                          */
typedef struct {
    int32_t n_req;
    int64_t n_total;
    const int64_t *req_off;
    const int32_t *block_table;
    int32_t max_pages;
} kvs_batch;

/* fp32 [max_pos][head_dim/2] tables of cos/sin(p * theta^(-2i/d)). */
typedef struct {
    const float *cos;
    const float *sin;
    int32_t max_pos;
} kvs_rope;

/* G1: for every flat position t with src_slot[t] >= 0, copy K and V rows of
 * layers [layer_begin, layer_end) from slot page slot_pages[slot*slot_max_pages
 * + cand/page] into the request's page, rotating K by (pos - cand) when
 * rope != NULL.  Reused positions are found from the hit map itself.        */
kvs_status kvs_gather_kv(const kvs_kv_arena *arena, const kvs_batch *batch,
                         const int32_t *src_slot, const int32_t *src_cand,
                         const int32_t *slot_pages, int32_t slot_max_pages,
                         int32_t layer_begin, int32_t layer_end, const kvs_rope *rope,
                         kvs_stream_t stream);
/* G1 over a sharded pool with peer memory (multi-GPU): slot s is
 * owned by GPU slot_owner[s] (-1 = this GPU) and its pages (slot_pages, in the
 * owner's page numbering) are read from peer_base[owner], the owner's arena
 * base mapped into this process (CUDA IPC; NVLink loads between GPUs).  The
 * remote-shard fetch and the gather with RoPE re-alignment are one kernel -
 * the peer-memory alternative to the kvs_pack_rows / exchange /
 * kvs_unpack_rows path.  Replaces the same reference code as kvs_gather_kv
 * plus the cross-GPU read of the pool (simulate.py:182-189 reads one shared
 * pool).  slot_owner: int32 [n_slots]; peer_base: uint64 [world] (device). */
kvs_status kvs_gather_kv_peer(const kvs_kv_arena *arena, const kvs_batch *batch,
                              const int32_t *src_slot, const int32_t *src_cand,
                              const int32_t *slot_pages, int32_t slot_max_pages,
                              const int32_t *slot_owner, const uint64_t *peer_base,
                              int32_t layer_begin, int32_t layer_end, const kvs_rope *rope,
                              kvs_stream_t stream);

/* X1 remote-shard fetch (multi-GPU).  The owner packs the rows
 * (slot, cand) a peer hit - all layers, K and V - into a dense buffer
 * [n_rows][L][2][kv_heads*head_dim] bf16 that travels over NCCL send/recv;
 * the requester unpacks layers [layer_begin, layer_end) of them into its
 * pages at flat positions flat_t, re-aligning K by (pos - cand) like
 * kvs_gather_kv; rows whose skip[flat_t] (nullable, u8) is set are left
 * alone (the fast prefill path restores cached layer-0 rows only for the
 * reused positions DHD did not select).                                   */
kvs_status kvs_pack_rows(const kvs_kv_arena *arena, const int32_t *slot, const int32_t *cand,
                         int64_t n_rows, const int32_t *slot_pages, int32_t slot_max_pages,
                         void *out, kvs_stream_t stream);
kvs_status kvs_unpack_rows(const kvs_kv_arena *arena, const kvs_batch *batch,
                           const int64_t *flat_t, const int32_t *cand, int64_t n_rows,
                           const void *in, const kvs_rope *rope, int32_t layer_begin,
                           int32_t layer_end, const uint8_t *skip, kvs_stream_t stream);

/* F4 comparison strategies (selection.py:133-186).
 * kvs_topk_select: per request r (positions [req_off[r], req_off[r+1]),
 *   length <= max_len <= 47104), selected[t] = 1 for the budget[r] candidates
 *   (cand[t] >= 0) with the largest scores[t] >= 0, ties to the lower
 *   position (_take_top, selection.py:63-66).
 * kvs_ideal_scores: IDEAL leave-one-in scores (selection.py:172-183):
 *   scores[i] = ||attn(q, k + e_i dk, v + e_i dv) - attn(q, k, v)||_F over
 *   heads, rows and dims; q [H][n][d], k/v/dk/dv [kv_heads][n][d] fp32
 *   (GQA: query head h uses kv head h / (H / kv_heads)), d <= 256.        */
kvs_status kvs_topk_select(const float *scores, const int32_t *cand, const int64_t *req_off,
                           int32_t n_req, int64_t max_len, const int32_t *budget,
                           uint8_t *selected, kvs_stream_t stream);
size_t kvs_ideal_scores_workspace(int32_t num_heads, int32_t n, int32_t d);
kvs_status kvs_ideal_scores(const float *q, const float *k, const float *v, const float *dk,
                            const float *dv, int32_t num_heads, int32_t kv_heads, int32_t n,
                            int32_t d, int32_t causal, float softmax_scale, float *scores,
                            void *ws, size_t ws_bytes, kvs_stream_t stream);

/* F3/F1 pool-entry transfer (reference pool.py:100-123, 174-241): an entry's
 * K and V as dense fp32 [num_layers][n_tokens][kv_heads][d_k] - the KVSH file
 * order - to (import) or from (export) its arena pages (pages[i] holds tokens
 * [i*page_size, (i+1)*page_size)).  Import rounds to bf16 (RNE) and zeroes
 * the padded head lanes; export is exact.  k/v are device pointers.        */
kvs_status kvs_entry_import(const kvs_kv_arena *arena, const int32_t *pages, int64_t n_tokens,
                            int32_t d_k, const float *k, const float *v, kvs_stream_t stream);
kvs_status kvs_entry_export(const kvs_kv_arena *arena, const int32_t *pages, int64_t n_tokens,
                            int32_t d_k, float *k, float *v, kvs_stream_t stream);

/* Post-GEMM step for a set of query rows: qkv[row] = [q (H*d) | k (kvh*d) | v (kvh*d)]
 * bf16.  Rotates q,k by position (rope nullable), writes q to q_out[row][H][d],
 * writes k,v into the arena at (row_req, row_pos, layer) when write_kv[row]
 * != 0, and optionally dense copies k_out/v_out[row][kvh][d] (nullable).
 * q_out == NULL skips the query heads (kvs_attention_fwd_qkv rotates them). */
kvs_status kvs_qkv_rope_scatter(const void *qkv, int64_t n_rows, int32_t num_heads,
                                const int32_t *row_req, const int32_t *row_pos,
                                const uint8_t *write_kv, int32_t layer,
                                const kvs_kv_arena *arena, const kvs_batch *batch,
                                const kvs_rope *rope, void *q_out, void *k_out, void *v_out,
                                kvs_stream_t stream);
/* Same, reading output row i's q|k|v from qkv[src_row[i]] (head_dim 128):
 * the partial prefill's first session layer takes its rows of the probe's
 * all-row projection instead of projecting them again.                     */
kvs_status kvs_qkv_rope_scatter_rows(const void *qkv, const int32_t *src_row, int64_t n_rows,
                                     int32_t num_heads, const int32_t *row_req,
                                     const int32_t *row_pos, const uint8_t *write_kv,
                                     int32_t layer, const kvs_kv_arena *arena,
                                     const kvs_batch *batch, const kvs_rope *rope, void *q_out,
                                     void *k_out, void *v_out, kvs_stream_t stream);

/* Embedding rows: out[r] = table[ids[rows ? rows[r] : r]] (width bf16 each);
 * out_f32 (nullable) receives the same rows widened to fp32 (the residual
 * stream, model.py:189 embed). */
kvs_status kvs_embed_rows(const void *table, int64_t width, const int64_t *ids,
                          const int32_t *rows, int64_t n_rows, void *out, float *out_f32,
                          kvs_stream_t stream);

/* Decode-size projection (1 <= m <= 64 rows; model.py:193-195 / :202):
 * out = x @ W for W [k][n] bf16 given packed as 16 x 64 tiles of its
 * transpose, w_p [n/16][k/64][16][64] (W[i][j] at [j/16][i/64][j%16][i%64]),
 * x [m][k] bf16; n % 128 == 0, k % 512 == 0.  accumulate == 0: out is bf16
 * [m][n] and out_bf16 must be NULL.  accumulate != 0: out is fp32 [m][n] and
 * receives out += x @ W (the residual add); out_bf16 (nullable) then gets
 * bf16(out), the next layer's projection operand.  Deterministic (fixed
 * summation order).  Replaces the library GEMM of engine.py's decode steps. */
kvs_status kvs_proj_skinny(const void *x, int64_t m, const void *w_p, int64_t n, int64_t k,
                           int32_t accumulate, void *out, void *out_bf16, kvs_stream_t stream);

/* Recompute row set S = non-reused U selected U {n-1} per request (the rows a
 * partial prefill must compute).  Call once with
 * row_tok == NULL to get counts[r]; then with row_off[r] (exclusive prefix of
 * counts) to emit rows in position order: flat token index, request,
 * position, and write_kv = 1 when the row's K/V are recomputed (non-reused or
 * selected), 0 for a reused-unselected last row.  selected may be NULL.    */
kvs_status kvs_build_rows(const int64_t *req_off, int32_t n_req, const int32_t *src_slot,
                          const uint8_t *selected, int32_t *counts, const int64_t *row_off,
                          int32_t *row_tok, int32_t *row_req, int32_t *row_pos, uint8_t *write_kv,
                          kvs_stream_t stream);

/* ------------------------------------------------------------------ attention
 * Query rows are grouped into tiles of <= 128 rows of ONE request with
 * ascending positions: tile_req[t], tile_row0[t] (first row in q), tile_rows[t].
 * Row r attends keys [0, row_pos[r]] of its request (position-causal,
 * model.py:103-104) when causal != 0, else keys [0, kv_len[req]).
 * q, out: [n_rows][num_heads][head_dim] bf16; lse (nullable): [n_rows][H] f32
 * natural-log softmax normaliser.  head_dim must be 128.                    */
kvs_status kvs_attention_fwd(const void *q, const int32_t *row_pos, int64_t n_rows,
                             int32_t num_heads, const int32_t *tile_req,
                             const int32_t *tile_row0, const int32_t *tile_rows,
                             int32_t n_tiles, const int32_t *kv_len, int32_t causal,
                             int32_t layer, const kvs_kv_arena *arena, const kvs_batch *batch,
                             float softmax_scale, void *out, float *lse, kvs_stream_t stream);

/* kvs_attention_fwd with the query rows read straight from the QKV
 * projection: qkv[row][qkv_row_stride] bf16 whose first num_heads*128
 * elements are the UN-rotated query heads; the kernel rotates each Q tile
 * by row_pos in shared memory (rope nullable: no rotation) before the first
 * Q.K^T, bit-identical to kvs_qkv_rope_scatter's rotation, so a caller can
 * skip writing q (kvs_qkv_rope_scatter with q_out == NULL).  Replaces the
 * same reference code as kvs_attention_fwd (model.py:110-129, 193-195, 201);
 * even GQA groups and odd groups (the fwd3 / fwd6 kernels) only.          */
kvs_status kvs_attention_fwd_qkv(const void *qkv, int64_t qkv_row_stride, const kvs_rope *rope,
                                 const int32_t *row_pos, int64_t n_rows, int32_t num_heads,
                                 const int32_t *tile_req, const int32_t *tile_row0,
                                 const int32_t *tile_rows, int32_t n_tiles,
                                 const int32_t *kv_len, int32_t causal, int32_t layer,
                                 const kvs_kv_arena *arena, const kvs_batch *batch,
                                 float softmax_scale, void *out, kvs_stream_t stream);

/* Few-row attention (decode steps, probe queries): same semantics as
 * kvs_attention_fwd for arbitrary rows (row_req per row; rows of one request
 * contiguous), split-K flash decoding on mma.sync tiles where a request's rows
 * share every K/V page; num_heads / kv_heads <= 8, page_size 64.  The
 * workspace starts with 256 KB of split counters that must be zero when the
 * buffer is first used; every call leaves them zero again.                */
size_t kvs_decode_attention_workspace(int64_t n_rows, int32_t num_heads, int32_t kv_heads,
                                      int32_t head_dim, int32_t max_kv);
kvs_status kvs_decode_attention(const void *q, const int32_t *row_req, const int32_t *row_pos,
                                int64_t n_rows, int32_t num_heads, const int32_t *kv_len,
                                int32_t causal, int32_t layer, const kvs_kv_arena *arena,
                                const kvs_batch *batch, float softmax_scale, void *out,
                                void *ws, size_t ws_bytes, kvs_stream_t stream);

/* ------------------------------------------------------------------ DHD
 * D1: alpha[t] = (1/H) * sum_h sum_{j >= i} softmax_j(q_j . k_i * scale)[i]
 * for each request's rows t = position i (q dense [n_total][H][128], row t
 * of the batch = position row_pos[t]; K = the arena's `layer`).  Rows are
 * tiled like kvs_attention_fwd (tiles of <= 128 consecutive positions of one
 * request).  Two tcgen05 passes: row log-sum-exp, then key-major column sums.
 * causal == 0 sums over all rows (kv_len[r] = request length).            */
size_t kvs_dhd_alpha_workspace(int64_t n_total, int32_t num_heads, int32_t kv_heads);
kvs_status kvs_dhd_alpha(const void *q, int32_t num_heads, int32_t causal, int32_t layer,
                         const kvs_kv_arena *arena, const kvs_batch *batch,
                         const int32_t *row_pos, const int32_t *tile_req,
                         const int32_t *tile_row0, const int32_t *tile_rows, int32_t n_tiles,
                         const int32_t *kv_len, float softmax_scale, float *alpha, void *ws,
                         size_t ws_bytes, kvs_stream_t stream);

/* D2: for every reused flat position t (src_slot[t] >= 0):
 *   dv_l1[t] = sum_{g,i} |V_arena(layer)[t] - v_true[t]|, score[t] = alpha[t]*dv_l1[t]
 * then per request keep budget[r] reused positions by (score desc, pos asc)
 * (selection.py:63-66); selected[t] = 1 for kept positions.  Non-reused
 * positions get score 0 and selected 0.  budget is host-computed with the
 * reference's IEEE-double ceil (selection.py:51-52).  One launch for the
 * whole batch.  Workspace: kvs_dhd_select_workspace(n_total, n_req) bytes
 * (self-resetting counters, then one 32-bit selection key per position);
 * its first 256 bytes must be zero before the first call on a buffer and
 * are left zero by every call.                                              */
size_t kvs_dhd_select_workspace(int64_t n_total, int32_t n_req);
kvs_status kvs_dhd_select(const void *v_true, const float *alpha, const int32_t *src_slot,
                          int32_t layer, const kvs_kv_arena *arena, const kvs_batch *batch,
                          const int32_t *budget, float *dv_l1, float *score,
                          uint8_t *selected, void *ws, size_t ws_bytes, kvs_stream_t stream);

/* D3: one decode step per request r: w_i = mean_h softmax_i(q_t[r,h] . K_i /
 * sqrt(d)) over ALL ctx_len[r] rows of the arena's `layer` (no mask,
 * selection.py:100-103), score_i = w_i * dv_l1[r-th prefill row i]; choose
 * min(n_extra, #eligible) eligible rows by (score desc, pos asc).
 * eligible: flat [n_total] u8 over each request's prefill rows (updated in
 * place: chosen rows cleared); chosen: [n_req][n_extra] int32 ascending,
 * n_chosen: [n_req]; scores (nullable): [n_req][max_ctx] f32.
 * One fused persistent cooperative launch (page_size 64, head_dim 128, n_extra <= 16,
 * num_heads <= 64 and even, n_req <= 1024; else a two-kernel fallback).  Workspace:
 * kvs_dhd_decode_select_workspace() bytes whose first 4352 bytes (a counter
 * header of one fixed size: work ticket, grid barrier and per-request
 * counters for up to 1024 requests) must be zero before the first call on a
 * buffer and are left zero by every call, of any shape and on either path. */
size_t kvs_dhd_decode_select_workspace(int32_t n_req, int32_t num_heads, int32_t max_ctx);
kvs_status kvs_dhd_decode_select(const void *q_t, int32_t num_heads, const int32_t *ctx_len,
                                 int32_t max_ctx, const float *dv_l1, uint8_t *eligible,
                                 int32_t layer, const kvs_kv_arena *arena,
                                 const kvs_batch *batch, int32_t n_extra, float softmax_scale,
                                 int32_t *chosen, int32_t *n_chosen, float *scores, void *ws,
                                 size_t ws_bytes, kvs_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* KVSHARE_H_ */
