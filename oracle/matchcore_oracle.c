/*
 * TEST INFRASTRUCTURE ONLY - CPU oracle for the KV Retriever (parity checker).
 *
 * Plain-C restatement of the reference matcher and pool lookup, used only by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg.  The product path (paper_2503_16525_b200) never links or
 * calls this file.
 *
 * Follows, line for line in behaviour (not in code):
 *   window_hashes  - reference pkg/src/kvlab/_matchcore.pyx:16-34
 *                    (rolled polynomial hash, u64 arithmetic, m < 2^31)
 *   match_pairs    - reference pkg/src/kvlab/_matchcore.pyx:37-84
 *                    (stable hash index of the target, candidate windows j
 *                    ascending, bucket positions i ascending, token-equality
 *                    extension from k = 0, first claim wins, extension runs
 *                    through already-claimed positions)
 *   pool_lookup    - reference pkg/src/kvlab/pool.py:125-161
 *                    (entries newest-first, skip entries sharing no window
 *                    hash, first-come claims, early exit once every
 *                    position is claimed; contributor flags for the LRU
 *                    refresh at pool.py:157-159)
 *
 * Pinned against golden vectors produced by the reference itself
 * (tests/golden/make_golden.py) in tests/test_oracle_golden.py.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* Exact residue product.  The reference's compiled kernel requires
 * m < 2^31 (u64 products, matching.py:39-41, :110-113); beyond that its
 * pure backend is arbitrary precision, restated here with 128-bit products. */
static inline uint64_t mulmod(uint64_t a, uint64_t b, uint64_t m) {
    return (uint64_t)(((unsigned __int128)a * b) % m);
}

int64_t oracle_window_hashes(const int64_t *tok, int64_t n, int32_t w,
                             uint64_t b, uint64_t m, uint64_t *out) {
    if (n < w) return 0;
    uint64_t bw = 1;
    for (int32_t i = 0; i < w - 1; ++i) bw = mulmod(bw, b, m);
    uint64_t h = 0;
    for (int32_t i = 0; i < w; ++i) h = (mulmod(h, b, m) + ((uint64_t)tok[i]) % m) % m;
    out[0] = h;
    for (int64_t i = 1; i < n - w + 1; ++i) {
        uint64_t drop = mulmod(((uint64_t)tok[i - 1]) % m, bw, m);
        h = (mulmod((h + m - drop) % m, b, m) + ((uint64_t)tok[i + w - 1]) % m) % m;
        out[i] = h;
    }
    return n - w + 1;
}

typedef struct { uint64_t h; int64_t i; } hidx_t;

static int cmp_hidx(const void *a, const void *b) {
    const hidx_t *x = (const hidx_t *)a, *y = (const hidx_t *)b;
    if (x->h < y->h) return -1;
    if (x->h > y->h) return 1;
    return (x->i < y->i) ? -1 : (x->i > y->i);  /* stable: ascending position */
}

/* Returns the number of claimed pairs written to tm/cm (capacity >= nt). */
int64_t oracle_match_pairs(const int64_t *tgt, int64_t nt, const int64_t *cand,
                           int64_t nc, int32_t w, uint64_t b, uint64_t m,
                           int64_t *tm, int64_t *cm) {
    if (nt < w || nc < w) return 0;
    int64_t nth = nt - w + 1, nch = nc - w + 1;
    uint64_t *th = (uint64_t *)malloc(sizeof(uint64_t) * nth);
    uint64_t *ch = (uint64_t *)malloc(sizeof(uint64_t) * nch);
    hidx_t *idx = (hidx_t *)malloc(sizeof(hidx_t) * nth);
    uint8_t *matched = (uint8_t *)calloc((size_t)nt, 1);
    oracle_window_hashes(tgt, nt, w, b, m, th);
    oracle_window_hashes(cand, nc, w, b, m, ch);
    for (int64_t i = 0; i < nth; ++i) { idx[i].h = th[i]; idx[i].i = i; }
    qsort(idx, (size_t)nth, sizeof(hidx_t), cmp_hidx);
    int64_t count = 0;
    for (int64_t j = 0; j < nch; ++j) {
        uint64_t h = ch[j];
        int64_t lo = 0, hi = nth;
        while (lo < hi) {
            int64_t mid = (lo + hi) >> 1;
            if (idx[mid].h < h) lo = mid + 1; else hi = mid;
        }
        for (int64_t pos = lo; pos < nth && idx[pos].h == h; ++pos) {
            int64_t i = idx[pos].i;
            for (int64_t k = 0; i + k < nt && j + k < nc && tgt[i + k] == cand[j + k]; ++k) {
                if (!matched[i + k]) {
                    matched[i + k] = 1;
                    tm[count] = i + k;
                    cm[count] = j + k;
                    ++count;
                }
            }
        }
    }
    free(th); free(ch); free(idx); free(matched);
    return count;
}

/*
 * entries are given newest-first (insert_seq descending, pool.py:139).
 * entry_tokens: concatenated tokens, entry_off[e]..entry_off[e+1].
 * Outputs: src_entry[t] (index into the given order, -1 = miss),
 *          src_cand[t], contributed[e] (0/1).  Returns the hit count.
 */
int64_t oracle_pool_lookup(int32_t n_entries, const int64_t *entry_tokens,
                           const int64_t *entry_off, const int64_t *req, int64_t n,
                           int32_t w, uint64_t b, uint64_t m, int32_t *src_entry,
                           int32_t *src_cand, uint8_t *contributed) {
    for (int64_t t = 0; t < n; ++t) { src_entry[t] = -1; src_cand[t] = -1; }
    for (int32_t e = 0; e < n_entries; ++e) contributed[e] = 0;
    if (n == 0 || n_entries == 0) return 0;
    int64_t nth = n >= w ? n - w + 1 : 0;
    uint64_t *th = (uint64_t *)malloc(sizeof(uint64_t) * (nth ? nth : 1));
    oracle_window_hashes(req, n, w, b, m, th);
    /* sorted copy of the target hash set for the shared-hash prefilter */
    uint64_t *ths = (uint64_t *)malloc(sizeof(uint64_t) * (nth ? nth : 1));
    memcpy(ths, th, sizeof(uint64_t) * nth);
    hidx_t *tmp = (hidx_t *)malloc(sizeof(hidx_t) * (nth ? nth : 1));
    for (int64_t i = 0; i < nth; ++i) { tmp[i].h = ths[i]; tmp[i].i = i; }
    qsort(tmp, (size_t)nth, sizeof(hidx_t), cmp_hidx);
    for (int64_t i = 0; i < nth; ++i) ths[i] = tmp[i].h;
    free(tmp);
    int64_t *tm = (int64_t *)malloc(sizeof(int64_t) * n);
    int64_t *cm = (int64_t *)malloc(sizeof(int64_t) * n);
    int64_t hits = 0;
    for (int32_t e = 0; e < n_entries; ++e) {
        if (hits == n) break;                                   /* pool.py:142-143 */
        const int64_t *et = entry_tokens + entry_off[e];
        int64_t ne = entry_off[e + 1] - entry_off[e];
        /* pool.py:144-146: skip entries sharing no window hash */
        int shared = 0;
        if (ne >= w && nth > 0) {
            uint64_t *eh = (uint64_t *)malloc(sizeof(uint64_t) * (ne - w + 1));
            oracle_window_hashes(et, ne, w, b, m, eh);
            for (int64_t j = 0; j < ne - w + 1 && !shared; ++j) {
                int64_t lo = 0, hi = nth;
                while (lo < hi) {
                    int64_t mid = (lo + hi) >> 1;
                    if (ths[mid] < eh[j]) lo = mid + 1; else hi = mid;
                }
                shared = (lo < nth && ths[lo] == eh[j]);
            }
            free(eh);
        }
        if (!shared) continue;
        int64_t cnt = oracle_match_pairs(req, n, et, ne, w, b, m, tm, cm);
        for (int64_t p = 0; p < cnt; ++p) {
            int64_t t = tm[p];
            if (src_entry[t] < 0) {
                src_entry[t] = e;
                src_cand[t] = (int32_t)cm[p];
                contributed[e] = 1;
                ++hits;
            }
        }
    }
    free(th); free(ths); free(tm); free(cm);
    return hits;
}
