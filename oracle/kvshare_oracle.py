"""TEST INFRASTRUCTURE ONLY - CPU oracle for the KVShare DHD hot path.

This module is the parity checker.  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``) may import
it; the product package ``paper_2503_16525_b200`` never does, and it has no CPU
fallback that could route through here.

It restates the reference ``kvlab`` algorithms for the path in float64 numpy
(integer work in ``matchcore_oracle.c``), each function citing the reference
file:line it follows (paths relative to the reference's ``pkg/src/kvlab``).
Two extensions the reference lacks are restated so that they reduce exactly
to the reference when disabled:

* GQA (``num_kv_heads < num_heads``): query head ``h`` reads KV head
  ``h // (num_heads // num_kv_heads)``; DHD alpha is the mean over query heads,
  the value-deviation L1 norm is summed over KV heads.
* RoPE (``rope_theta`` not None): rotate-half rotary embedding of q and k by
  absolute position, using the fp32 cos/sin table from :func:`rope_table`;
  cached K rows are stored post-rotation at the entry's own positions and are
  re-aligned by a rotation of ``dst_pos - cand_pos``.

Pinning: tests/test_oracle_golden.py checks every function here against the
golden vectors produced by the reference itself (tests/golden/make_golden.py).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle_match.so")
_lib = None


def build_oracle(force: bool = False) -> str:
    """Compile the C restatement (gcc, -O2) into oracle/_build/."""
    src = os.path.join(_HERE, "matchcore_oracle.c")
    if force or not os.path.exists(_LIB_PATH) or \
            os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        os.makedirs(os.path.dirname(_LIB_PATH), exist_ok=True)
        subprocess.check_call(["gcc", "-O2", "-shared", "-fPIC", "-o", _LIB_PATH, src])
    return _LIB_PATH


def _c():
    global _lib
    if _lib is None:
        build_oracle()
        lib = ctypes.CDLL(_LIB_PATH)
        i64p = ctypes.POINTER(ctypes.c_int64)
        lib.oracle_window_hashes.restype = ctypes.c_int64
        lib.oracle_window_hashes.argtypes = [i64p, ctypes.c_int64, ctypes.c_int32,
                                             ctypes.c_uint64, ctypes.c_uint64,
                                             ctypes.POINTER(ctypes.c_uint64)]
        lib.oracle_match_pairs.restype = ctypes.c_int64
        lib.oracle_match_pairs.argtypes = [i64p, ctypes.c_int64, i64p, ctypes.c_int64,
                                           ctypes.c_int32, ctypes.c_uint64,
                                           ctypes.c_uint64, i64p, i64p]
        lib.oracle_pool_lookup.restype = ctypes.c_int64
        lib.oracle_pool_lookup.argtypes = [
            ctypes.c_int32, i64p, i64p, i64p, ctypes.c_int64, ctypes.c_int32,
            ctypes.c_uint64, ctypes.c_uint64, ctypes.POINTER(ctypes.c_int32),
            ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_uint8)]
        _lib = lib
    return _lib


def _i64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int64))


def _ptr(a, ctype):
    return a.ctypes.data_as(ctypes.POINTER(ctype))


# --------------------------------------------------------------------------
# KV Retriever (integer, bit-exact)
# --------------------------------------------------------------------------

def window_hashes(tokens, w: int = 8, b: int = 31, m: int = 1_000_000_007) -> np.ndarray:
    """_matchcore.pyx:16-34 / matching.py:135-142."""
    t = _i64(tokens)
    out = np.zeros(max(t.size - w + 1, 1), dtype=np.uint64)
    cnt = _c().oracle_window_hashes(_ptr(t, ctypes.c_int64), t.size, w, b, m,
                                    _ptr(out, ctypes.c_uint64))
    return out[:cnt]


def match_pairs(target, candidate, w: int = 8, b: int = 31, m: int = 1_000_000_007):
    """_matchcore.pyx:37-84 / matching.py:154-168: (target_matches, cand_matches)."""
    t, c = _i64(target), _i64(candidate)
    tm = np.zeros(max(t.size, 1), dtype=np.int64)
    cm = np.zeros(max(t.size, 1), dtype=np.int64)
    cnt = _c().oracle_match_pairs(_ptr(t, ctypes.c_int64), t.size, _ptr(c, ctypes.c_int64),
                                  c.size, w, b, m, _ptr(tm, ctypes.c_int64),
                                  _ptr(cm, ctypes.c_int64))
    return [int(x) for x in tm[:cnt]], [int(x) for x in cm[:cnt]]


def pool_lookup(entries_newest_first, request, w: int = 8, b: int = 31,
                m: int = 1_000_000_007):
    """pool.py:125-161.  ``entries_newest_first``: token arrays ordered by
    insert_seq descending.  Returns (src_entry[n], src_cand[n], contributed[E]);
    src_entry indexes the given order, -1 = miss."""
    req = _i64(request)
    toks = [_i64(e) for e in entries_newest_first]
    off = np.zeros(len(toks) + 1, dtype=np.int64)
    for i, e in enumerate(toks):
        off[i + 1] = off[i] + e.size
    flat = np.concatenate(toks) if toks else np.zeros(1, dtype=np.int64)
    flat = _i64(flat)
    n = req.size
    se = np.full(max(n, 1), -1, dtype=np.int32)
    sc = np.full(max(n, 1), -1, dtype=np.int32)
    contrib = np.zeros(max(len(toks), 1), dtype=np.uint8)
    _c().oracle_pool_lookup(len(toks), _ptr(flat, ctypes.c_int64), _ptr(off, ctypes.c_int64),
                            _ptr(req, ctypes.c_int64), n, w, b, m,
                            _ptr(se, ctypes.c_int32), _ptr(sc, ctypes.c_int32),
                            _ptr(contrib, ctypes.c_uint8))
    return se[:n], sc[:n], contrib[:len(toks)].astype(bool)


def fixed_chunk_lookup(entries_newest_first, request, chunk: int):
    """pool.py:139-159 with fixed_chunk -> matching.py:171-194, restated.
    Entries are visited newest first; each entry's fixed_chunk_match claims
    the still-unclaimed target chunks [i*c, (i+1)*c) for which the identical
    block sits at an aligned candidate offset j*c (first j wins; trailing
    partial chunks never match).  Returns (src_entry[n], src_cand[n],
    contributed[E]) like pool_lookup."""
    req = np.asarray(request, dtype=np.int64)
    n, c = req.size, int(chunk)
    se = np.full(n, -1, dtype=np.int32)
    sc = np.full(n, -1, dtype=np.int32)
    contrib = np.zeros(len(entries_newest_first), dtype=bool)
    for e, ent in enumerate(entries_newest_first):
        cand = np.asarray(ent, dtype=np.int64)
        blocks = [(j, cand[j:j + c]) for j in range(0, cand.size - c + 1, c)]
        for i in range(0, n - c + 1, c):
            for j, blk in blocks:
                if np.array_equal(req[i:i + c], blk):
                    if (se[i:i + c] < 0).any():
                        free = se[i:i + c] < 0
                        se[i:i + c][free] = e
                        sc[i:i + c][free] = np.arange(j, j + c)[free]
                        contrib[e] = True
                    break
    return se, sc, contrib


def hit_rate(n: int, n_hit: int) -> float:
    """matching.py:197-205 / pool.py:65-67."""
    return n_hit / n if n else 0.0


# --------------------------------------------------------------------------
# Scheduler hand-off (host logic)
# --------------------------------------------------------------------------

def schedule_order(hit_rates, arrivals, ids, batch_size: int, aging_lambda: float = 0.0,
                   now_ms: float = 0.0):
    """scheduling.py:106-125: stable sort by (-(h + lambda*wait), arrival, id),
    sliced into batches of <= batch_size; returns lists of indices."""
    eff = [h + aging_lambda * max(0.0, now_ms - a) for h, a in zip(hit_rates, arrivals)]
    order = sorted(range(len(ids)), key=lambda i: (-eff[i], arrivals[i], ids[i]))
    return [order[i:i + batch_size] for i in range(0, len(order), batch_size)]


# --------------------------------------------------------------------------
# Model restatement (float64)
# --------------------------------------------------------------------------

@dataclass(frozen=True)
class OracleConfig:
    num_layers: int = 4
    num_heads: int = 4
    d_model: int = 64
    vocab_size: int = 4096
    seed: int = 0
    num_kv_heads: int | None = None
    rope_theta: float | None = None

    @property
    def d_k(self) -> int:
        return self.d_model // self.num_heads

    @property
    def kvh(self) -> int:
        return self.num_kv_heads or self.num_heads

    @property
    def group(self) -> int:
        return self.num_heads // self.kvh


def draw_weights(cfg: OracleConfig) -> dict:
    """model.py:57-70: Philox(key=seed), uniform(-1,1)/sqrt(d_model), drawn in
    the order embedding, then per layer W_q, W_k, W_v, W_o.  With GQA, W_k/W_v
    are (d_model, kvh*d_k) (identical draws to the reference when kvh == H)."""
    gen = np.random.Generator(np.random.Philox(key=cfg.seed))
    scale = 1.0 / np.sqrt(cfg.d_model)

    def draw(rows, cols):
        return gen.uniform(-1.0, 1.0, size=(rows, cols)) * scale

    d, kvd = cfg.d_model, cfg.kvh * cfg.d_k
    emb = draw(cfg.vocab_size, d)
    layers = [(draw(d, d), draw(d, kvd), draw(d, kvd), draw(d, d))
              for _ in range(cfg.num_layers)]
    return {"embedding": emb, "layers": layers}


def rope_table(max_pos: int, d_k: int, theta: float):
    """fp32 cos/sin of angle p * theta^(-2i/d_k), p in [0, max_pos), i < d_k/2.
    The same table is uploaded to the GPU, so both sides rotate by identical
    coefficients."""
    inv = theta ** (-np.arange(0, d_k // 2, dtype=np.float64) * 2.0 / d_k)
    ang = np.arange(max_pos, dtype=np.float64)[:, None] * inv[None, :]
    return np.cos(ang).astype(np.float32), np.sin(ang).astype(np.float32)


def rotate(x: np.ndarray, delta, table) -> np.ndarray:
    """Rotate-half RoPE of rows x[..., n, d] by per-row integer angle index
    ``delta`` (may be negative: cos even, sin odd)."""
    cos_t, sin_t = table
    delta = np.asarray(delta, dtype=np.int64)
    c = cos_t[np.abs(delta)].astype(np.float64)
    s = sin_t[np.abs(delta)].astype(np.float64) * np.sign(delta)[:, None]
    half = x.shape[-1] // 2
    x1, x2 = x[..., :half], x[..., half:]
    return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1)


def split_heads(x, heads):
    """model.py:87-90."""
    n, dm = x.shape
    return x.reshape(n, heads, dm // heads).transpose(1, 0, 2)


def merge_heads(x):
    """model.py:93-96."""
    h, n, d = x.shape
    return x.transpose(1, 0, 2).reshape(n, h * d)


def softmax_rows(logits, causal=False):
    """model.py:99-107."""
    if causal:
        nq, nk = logits.shape[-2], logits.shape[-1]
        mask = np.triu(np.ones((nq, nk), dtype=bool), k=1)
        logits = np.where(mask, -np.inf, logits)
    shifted = logits - logits.max(axis=-1, keepdims=True)
    e = np.exp(shifted)
    return e / e.sum(axis=-1, keepdims=True)


def expand_kv(k, group):
    return np.repeat(k, group, axis=0) if group > 1 else k


# Above this many attention-matrix elements the restatement runs one query
# head at a time (same formula per element, bounded memory): Llama-width
# prefill at 4k-16k tokens would otherwise need (H, n, n) float64 temporaries
# of 4-60 GB.
_BIG = 1 << 25


def _heads_parallel(fn, H):
    """fn(h) for every head; numpy's BLAS and ufuncs release the GIL, so a
    thread pool spreads heads over the host cores."""
    from concurrent.futures import ThreadPoolExecutor
    workers = max(1, min(H, (os.cpu_count() or 1) // 2, 16))
    if workers == 1:
        return [fn(h) for h in range(H)]
    with ThreadPoolExecutor(workers) as ex:
        return list(ex.map(fn, range(H)))


def attention_rows(q, qpos, k, v, group=1):
    """model.py:110-129 for a subset of query rows: q (H, m, d) at absolute
    positions qpos[m], keys/values (kvh, n, d); key j is visible to a row at
    position p iff j <= p (softmax_rows' causal mask, model.py:102-104, read
    per row).  With qpos = arange(n) this is attention(q, k, v, causal=True).
    One head at a time; returns (H, m, d)."""
    H, m, d = q.shape
    n = k.shape[1]
    qpos = np.asarray(qpos, dtype=np.int64)
    hidden = np.arange(n)[None, :] > qpos[:, None]
    scale = 1.0 / math.sqrt(d)
    out = np.empty((H, m, v.shape[-1]))

    def one(h):
        g = h // group
        logits = q[h] @ k[g].T * scale
        logits[hidden] = -np.inf
        logits -= logits.max(axis=-1, keepdims=True)
        np.exp(logits, out=logits)
        logits /= logits.sum(axis=-1, keepdims=True)
        out[h] = logits @ v[g]

    _heads_parallel(one, H)
    return out


def attention(q, k, v, causal=True, group=1):
    """model.py:110-129 with GQA expansion: (H,n,d),(kvh,n,d) -> (H,n,d).
    Large causal problems go through attention_rows (attn is then None)."""
    if causal and q.ndim == 3 and q.shape[0] * q.shape[1] * k.shape[1] > _BIG:
        return attention_rows(q, np.arange(q.shape[1]), k, v, group), None
    k, v = expand_kv(k, group), expand_kv(v, group)
    attn = softmax_rows(q @ np.swapaxes(k, -1, -2) / math.sqrt(q.shape[-1]), causal=causal)
    return attn @ v, attn


def _qkv(x, w, cfg, table, positions):
    wq, wk, wv, _ = w
    q = split_heads(x @ wq, cfg.num_heads)
    k = split_heads(x @ wk, cfg.kvh)
    v = split_heads(x @ wv, cfg.kvh)
    if table is not None:
        q = rotate(q, positions, table)
        k = rotate(k, positions, table)
    return q, k, v


@dataclass
class Reuse:
    """Retriever output in array form: src_entry[n] (-1 = miss), src_cand[n],
    and the entries' cached K/V (L, kvh, n_e, d_k), K post-RoPE at the entry's
    own positions.  pool.py:58-75 (ReuseMap) restated."""
    src_entry: np.ndarray
    src_cand: np.ndarray
    entry_k: list
    entry_v: list

    @property
    def reused(self):
        return [int(p) for p in np.nonzero(self.src_entry >= 0)[0]]

    def cached_rows(self, layer, table):
        """Gather: model.py:196-200 / engine.py:204-206 (+ RoPE re-alignment)."""
        pos = np.array(self.reused, dtype=np.int64)
        if pos.size == 0:
            return pos, None, None
        kr = np.stack([self.entry_k[self.src_entry[p]][layer, :, self.src_cand[p], :]
                       for p in pos], axis=1)
        vr = np.stack([self.entry_v[self.src_entry[p]][layer, :, self.src_cand[p], :]
                       for p in pos], axis=1)
        if table is not None:
            kr = rotate(kr, pos - self.src_cand[pos], table)
        return pos, kr, vr


def forward(tokens, W, cfg: OracleConfig, reuse: Reuse | None = None,
            recompute=None, table=None):
    """model.py:163-208 (_forward): per layer QKV for all rows, cached K/V
    substituted at reused positions not in the layer's recompute set, causal
    attention over all n rows, residual.  Returns dict of stacked states."""
    tokens = np.asarray(tokens, dtype=np.int64)
    x = W["embedding"][tokens]
    n = x.shape[0]
    pos = np.arange(n)
    L = cfg.num_layers
    sets = [set()] * L if recompute is None else \
        [set(recompute.get(l, ())) if isinstance(recompute, dict) else set(recompute)
         for l in range(L)]
    qs, ks, vs, outs, hid = [], [], [], [], [x]
    for layer in range(L):
        w = W["layers"][layer]
        q, k, v = _qkv(x, w, cfg, table, pos)
        if reuse is not None:
            rpos, kr, vr = reuse.cached_rows(layer, table)
            for idx, p in enumerate(rpos):
                if p in sets[layer]:
                    continue
                k[:, p, :] = kr[:, idx, :]
                v[:, p, :] = vr[:, idx, :]
        out, _ = attention(q, k, v, causal=True, group=cfg.group)
        x = x + merge_heads(out) @ w[3]
        qs.append(q); ks.append(k); vs.append(v); outs.append(out); hid.append(x)
    return {"q": np.stack(qs), "k": np.stack(ks), "v": np.stack(vs),
            "head_out": np.stack(outs), "hidden": np.stack(hid)}


def partial_rows(n, reused, selected):
    """SURVEY.md A12 row set S = non-reused U selected U {n-1}, ascending."""
    keep = np.ones(n, dtype=bool)
    keep[list(reused)] = False
    keep[list(selected)] = True
    keep[n - 1] = True
    return np.nonzero(keep)[0]


def forward_rows(tokens, W, cfg: OracleConfig, reuse: Reuse | None, selected, rows=None,
                 table=None):
    """model.py:163-208 (_forward with one recompute set at every layer,
    engine.py:241) computing query rows ``rows`` only - by default the row
    set S of :func:`partial_rows`.  Every row whose K/V is fresh (non-reused
    or selected) must be in ``rows``: then the K/V caches are complete and the
    hidden states of the computed rows equal the full forward's rows
    (verified 0.0 difference; pinned here by
    tests/test_oracle_golden.py against the reference's own prefill states).

    Returns {"rows": rows, "hidden": (L+1, m, d_model) for those rows,
    "k"/"v": (L, kvh, n, d_k) complete caches}."""
    tokens = np.asarray(tokens, dtype=np.int64)
    n = tokens.size
    reused = reuse.reused if reuse is not None else []
    selected = sorted(set(int(s) for s in selected))
    rows = partial_rows(n, reused, selected) if rows is None else \
        np.asarray(sorted(set(int(r) for r in rows)), dtype=np.int64)
    fresh = np.ones(n, dtype=bool)
    fresh[reused] = False
    fresh[selected] = True
    in_rows = np.zeros(n, dtype=bool)
    in_rows[rows] = True
    if (fresh & ~in_rows).any():
        raise ValueError("every fresh (non-reused or selected) row must be computed")
    write = fresh[rows]
    x = W["embedding"][tokens[rows]]
    hid, ks, vs = [x], [], []
    for layer in range(cfg.num_layers):
        w = W["layers"][layer]
        q, k_r, v_r = _qkv(x, w, cfg, table, rows)
        K = np.zeros((cfg.kvh, n, k_r.shape[-1]))
        V = np.zeros_like(K)
        if reuse is not None and reused:
            rpos, kr, vr = reuse.cached_rows(layer, table)
            K[:, rpos], V[:, rpos] = kr, vr
        K[:, rows[write]] = k_r[:, write]
        V[:, rows[write]] = v_r[:, write]
        out = attention_rows(q, rows, K, V, cfg.group)
        x = x + merge_heads(out) @ w[3]
        hid.append(x)
        ks.append(K)
        vs.append(V)
    return {"rows": rows, "hidden": np.stack(hid), "k": np.stack(ks), "v": np.stack(vs)}


def exact_hidden_at(tokens, W, cfg, layer, table=None):
    """engine.py:182-192."""
    tokens = np.asarray(tokens, dtype=np.int64)
    x = W["embedding"][tokens]
    pos = np.arange(x.shape[0])
    for l in range(layer):
        w = W["layers"][l]
        q, k, v = _qkv(x, w, cfg, table, pos)
        out, _ = attention(q, k, v, causal=True, group=cfg.group)
        x = x + merge_heads(out) @ w[3]
    return x


def perturbed_probe(tokens, W, cfg, reuse: Reuse, probe, table=None):
    """engine.py:195-207: probe-layer q, exact k/v and cache-substituted k/v."""
    x = exact_hidden_at(tokens, W, cfg, probe, table)
    q, kt, vt = _qkv(x, W["layers"][probe], cfg, table, np.arange(x.shape[0]))
    kp, vp = kt.copy(), vt.copy()
    rpos, kr, vr = reuse.cached_rows(probe, table)
    if rpos.size:
        kp[:, rpos, :] = kr
        vp[:, rpos, :] = vr
    return q, kt, vt, kp, vp


def v_impact_scores(q, k, delta_v, causal=True, group=1):
    """deviation.py:96-115 (+GQA): colsum of causal softmax averaged over query
    heads, times the L1 norm of delta_v summed over (kv) heads."""
    q, k, dv = np.asarray(q, float), np.asarray(k, float), np.asarray(delta_v, float)
    if causal and q.ndim == 3 and q.shape[0] * q.shape[1] * k.shape[1] > _BIG:
        return _alpha_per_head(q, k, group) * np.abs(dv).sum(axis=-1).sum(axis=0)
    kk = expand_kv(k, group) if k.ndim == 3 else k
    attn = softmax_rows(q @ np.swapaxes(kk, -1, -2) / math.sqrt(q.shape[-1]), causal=causal)
    alpha = attn.sum(axis=-2)
    l1 = np.abs(dv).sum(axis=-1)
    if attn.ndim == 3:
        alpha = alpha.mean(axis=0)
        l1 = l1.sum(axis=0)
    return alpha * l1


def _alpha_per_head(q, k, group):
    """deviation.py:108-110 (causal column sums of the softmax, mean over
    query heads) one head at a time, for problems too large for (H, n, n)."""
    H, n, d = q.shape
    hidden = np.triu(np.ones((n, n), dtype=bool), k=1)
    scale = 1.0 / math.sqrt(d)

    def one(h):
        logits = q[h] @ k[h // group].T * scale
        logits[hidden] = -np.inf
        logits -= logits.max(axis=-1, keepdims=True)
        np.exp(logits, out=logits)
        logits /= logits.sum(axis=-1, keepdims=True)
        return logits.sum(axis=0)

    return np.mean(_heads_parallel(one, H), axis=0)


def dhd_alpha(q, k, causal=True, group=1):
    """The alpha half of v_impact_scores (deviation.py:108-110)."""
    if causal and q.ndim == 3 and q.shape[0] * q.shape[1] * k.shape[1] > _BIG:
        return _alpha_per_head(q, k, group)
    kk = expand_kv(k, group) if k.ndim == 3 else k
    attn = softmax_rows(q @ np.swapaxes(kk, -1, -2) / math.sqrt(q.shape[-1]), causal=causal)
    alpha = attn.sum(axis=-2)
    return alpha.mean(axis=0) if attn.ndim == 3 else alpha


def budget(ratio: float, n_reused: int) -> int:
    """selection.py:51-52 - exact IEEE-double ceil."""
    return min(math.ceil(ratio * n_reused), n_reused)


def take_top(scores, eligible, count):
    """selection.py:63-66."""
    ranked = sorted(eligible, key=lambda i: (-scores[i], i))
    return tuple(sorted(ranked[:count]))


def select_prefill(q, k, delta_v, reused, ratio, causal=True, group=1):
    """selection.py:69-77."""
    reused = sorted(set(int(i) for i in reused))
    scores = v_impact_scores(q, k, delta_v, causal=causal, group=group)
    return take_top(scores, reused, budget(ratio, len(reused))), scores


def _spans(positions):
    runs = []
    for p in positions:
        if runs and p == runs[-1][-1] + 1:
            runs[-1].append(p)
        else:
            runs.append([p])
    return runs


def select_baseline(strategy, q, k, v, dk, dv, reused, ratio, seed=0, causal=True, group=1):
    """selection.py:133-186 restated for the comparison strategies.
    Returns (indices tuple, scores[n]).  IDEAL is the reference's literal
    leave-one-in loop (one attention pass per reused position)."""
    reused = sorted(set(int(i) for i in reused))
    q, k, v, dk, dv = (np.asarray(x, float) for x in (q, k, v, dk, dv))
    if q.ndim == 2:
        q, k, v, dk, dv = (x[None] for x in (q, k, v, dk, dv))
    n = k.shape[1]
    b = budget(ratio, len(reused))
    if strategy == "attention_weighted":
        return select_prefill(q, k + dk, dv, reused, ratio, causal=causal, group=group)
    if strategy == "magnitude":
        scores = np.abs(dv).sum(axis=(0, 2)) + np.abs(dk).sum(axis=(0, 2))
        return take_top(scores, reused, b), scores
    if strategy == "positional":
        chosen = []
        for span in _spans(reused):
            chosen.extend(span[: math.ceil(ratio * len(span))])
        if len(chosen) > b:
            chosen = sorted(chosen)[:b]
        elif len(chosen) < b:
            taken = set(chosen)
            chosen.extend([p for p in reused if p not in taken][: b - len(chosen)])
        return tuple(sorted(chosen)), np.zeros(n)
    if strategy == "random":
        gen = np.random.Generator(np.random.Philox(key=seed))
        scores = np.zeros(n)
        scores[reused] = gen.uniform(size=len(reused))
        return take_top(scores, reused, b), scores
    if strategy == "ideal":
        base, _ = attention(q, k, v, causal=causal, group=group)
        scores = np.zeros(n)
        for i in reused:
            k1, v1 = k.copy(), v.copy()
            k1[:, i, :] += dk[:, i, :]
            v1[:, i, :] += dv[:, i, :]
            pert, _ = attention(q, k1, v1, causal=causal, group=group)
            scores[i] = np.linalg.norm(pert - base)
        return take_top(scores, reused, b), scores
    raise ValueError(f"unknown strategy {strategy!r}")


def oracle_prefill(tokens, W, cfg, reuse, strategy, ratio, ref_states, table=None, seed=0):
    """engine.py:245-285 ORACLE mode restated: per layer, fresh q/k/v for all
    rows, cached rows substituted (k_pert, v_pert), deviations against the
    reference pass's k/v restricted to the reused rows, select_baseline on
    them, the layer's selected rows restored to fresh, attention, residual.
    Returns (sets per layer, hidden (L+1, n, d_model))."""
    tokens = np.asarray(tokens, dtype=np.int64)
    x = W["embedding"][tokens]
    n = x.shape[0]
    pos = np.arange(n)
    reused = reuse.reused
    keep = np.zeros(n, bool)
    keep[reused] = True
    sets, hid = [], [x]
    for layer in range(cfg.num_layers):
        w = W["layers"][layer]
        q, k_fresh, v_fresh = _qkv(x, w, cfg, table, pos)
        kp, vp = k_fresh.copy(), v_fresh.copy()
        rpos, kr, vr = reuse.cached_rows(layer, table)
        for idx, p in enumerate(rpos):
            kp[:, p, :] = kr[:, idx, :]
            vp[:, p, :] = vr[:, idx, :]
        dk = (kp - ref_states["k"][layer]) * keep[None, :, None]
        dv = (vp - ref_states["v"][layer]) * keep[None, :, None]
        idx, _ = select_baseline(strategy, q, ref_states["k"][layer], ref_states["v"][layer],
                                 dk, dv, reused, ratio, seed=seed, group=cfg.group)
        for p in idx:
            kp[:, p, :] = k_fresh[:, p, :]
            vp[:, p, :] = v_fresh[:, p, :]
        sets.append(set(idx))
        out, _ = attention(q, kp, vp, causal=True, group=cfg.group)
        x = x + merge_heads(out) @ w[3]
        hid.append(x)
    return sets, np.stack(hid)


def select_decode_step(q_t, k, delta_v, eligible, n_extra, group=1):
    """selection.py:80-105 (+GQA): unmasked softmax over the whole context,
    mean over query heads, times the delta_v L1 summed over kv heads."""
    q_t = np.atleast_2d(np.asarray(q_t, float))
    k = np.asarray(k, float)
    dv = np.asarray(delta_v, float)
    if k.ndim == 2:
        k, dv = k[None], dv[None]
    n = k.shape[1]
    eligible = sorted(set(int(i) for i in eligible))
    if not eligible or n_extra <= 0:
        return (), np.zeros(n)
    kk = expand_kv(k, group)
    logits = np.einsum("hd,hnd->hn", q_t, kk) / math.sqrt(q_t.shape[-1])
    weights = softmax_rows(logits).mean(axis=0)
    scores = weights * np.abs(dv).sum(axis=-1).sum(axis=0)
    return take_top(scores, eligible, min(n_extra, len(eligible))), scores


def restrict_rows(delta, keep):
    """engine.py:210-214."""
    out = np.zeros_like(delta)
    idx = sorted(keep)
    out[:, idx, :] = delta[:, idx, :]
    return out


def prefill_with_selection(tokens, W, cfg, reuse: Reuse, ratio, table=None):
    """engine.py:217-243 (PRACTICAL, ATTENTION_WEIGHTED via selection.py:156):
    probe = layer 1 (0 if L == 1), select, then the reuse forward with the same
    recompute set at every layer.  Returns (states, selected, eligible, probe)."""
    reused = reuse.reused
    if not reused:
        return forward(tokens, W, cfg, None, None, table), (), set(), None
    probe = 1 if cfg.num_layers >= 2 else 0
    q, kt, vt, kp, vp = perturbed_probe(tokens, W, cfg, reuse, probe, table)
    dk = restrict_rows(kp - kt, set(reused))
    dv = restrict_rows(vp - vt, set(reused))
    selected, scores = select_prefill(q, kt + dk, dv, reused, ratio, group=cfg.group)
    states = forward(tokens, W, cfg, reuse, {l: set(selected) for l in range(cfg.num_layers)},
                     table)
    info = {"q": q, "k_pert": kt + dk, "dv": dv, "scores": scores, "probe": probe}
    return states, selected, set(reused) - set(selected), info


def _one_row_attention(q, keys, vals, group):
    """engine.py:104-109: one query row per head over the whole given
    context (no mask), GQA heads grouped instead of expanded: q (H, d),
    keys/vals (kvh, n, d) -> (H, d)."""
    kvh, n, d = keys.shape
    qg = q.reshape(kvh, group, d)
    logits = np.einsum("gjd,gnd->gjn", qg, keys) / math.sqrt(d)
    wts = softmax_rows(logits)
    return np.einsum("gjn,gnd->gjd", wts, vals).reshape(kvh * group, d)


class Session:
    """engine.py:47-171 (ReuseSession) restated over numpy arrays: growing
    per-layer K/V cache (L, kvh, n, d), append / recompute_positions /
    query_rows_probe / delta_v_probe."""

    def __init__(self, tokens, W, cfg, states, reused=(), recomputed=(), table=None):
        self.W, self.cfg, self.table = W, cfg, table
        self.tokens = [int(t) for t in tokens]
        self.n_prefill = len(self.tokens)
        self.k = states["k"].copy()
        self.v = states["v"].copy()
        self.reused = set(reused)
        self.recomputed = [set(recomputed) & self.reused for _ in range(cfg.num_layers)]
        self.probe_layer = 1 if cfg.num_layers >= 2 else 0
        self._truth = None

    def probe_truth(self):
        """engine.py:81-89."""
        if self._truth is None:
            x = exact_hidden_at(self.tokens[:self.n_prefill], self.W, self.cfg,
                                self.probe_layer, self.table)
            self._truth = split_heads(x @ self.W["layers"][self.probe_layer][2], self.cfg.kvh)
        return self._truth

    def _token_rows(self, token_id, context):
        """engine.py:91-112."""
        cfg, W = self.cfg, self.W
        h = W["embedding"][token_id]
        p = context - 1
        for layer, w in enumerate(W["layers"]):
            q, k_new, v_new = _qkv(h[None], w, cfg, self.table, np.array([p]))
            self.k[layer, :, p, :] = k_new[:, 0, :]
            self.v[layer, :, p, :] = v_new[:, 0, :]
            out = _one_row_attention(q[:, 0, :], self.k[layer, :, :context, :],
                                     self.v[layer, :, :context, :], cfg.group)
            h = h + out.reshape(-1) @ w[3]
        return h

    def append(self, token_id):
        """engine.py:114-121."""
        L, kvh, _, d = self.k.shape
        pad = np.zeros((L, kvh, 1, d))
        self.k = np.concatenate([self.k, pad], axis=2)
        self.v = np.concatenate([self.v, pad], axis=2)
        self.tokens.append(int(token_id))
        return self._token_rows(int(token_id), len(self.tokens))

    def recompute_positions(self, positions):
        """engine.py:123-138."""
        for pos in sorted(set(int(p) for p in positions)):
            self._token_rows(self.tokens[pos], pos + 1)
            if pos in self.reused:
                for s in self.recomputed:
                    s.add(pos)

    def delta_v_probe(self):
        """engine.py:140-148."""
        delta = np.zeros_like(self.v[self.probe_layer])
        n = self.n_prefill
        delta[:, :n, :] = self.v[self.probe_layer, :, :n, :] - self.probe_truth()
        return delta

    def query_rows_probe(self, token_id):
        """engine.py:150-171."""
        cfg, W = self.cfg, self.W
        h = W["embedding"][token_id]
        p = len(self.tokens)
        for layer in range(self.probe_layer):
            w = W["layers"][layer]
            q, k_new, v_new = _qkv(h[None], w, cfg, self.table, np.array([p]))
            out = _one_row_attention(q[:, 0, :], np.concatenate([self.k[layer], k_new], axis=1),
                                     np.concatenate([self.v[layer], v_new], axis=1), cfg.group)
            h = h + out.reshape(-1) @ w[3]
        q, _, _ = _qkv(h[None], W["layers"][self.probe_layer], cfg, self.table, np.array([p]))
        return q[:, 0, :]


def run_generation(session: Session, decode_tokens, n_extra, eligible=None):
    """engine.py:298-328 without the reference-session metric: returns the
    chosen positions per step and the final-layer output row per step."""
    if eligible is None:
        eligible = set(session.reused) - set.intersection(*session.recomputed) \
            if session.recomputed else set(session.reused)
    eligible = set(eligible)
    chosen_steps, outs = [], []
    for tok in decode_tokens:
        chosen = ()
        if n_extra > 0 and eligible:
            q_t = session.query_rows_probe(int(tok))
            chosen, _ = select_decode_step(q_t, session.k[session.probe_layer],
                                           session.delta_v_probe(), eligible, n_extra,
                                           group=session.cfg.group)
            if chosen:
                session.recompute_positions(chosen)
                eligible -= set(chosen)
        outs.append(session.append(int(tok)))
        chosen_steps.append(chosen)
    return chosen_steps, outs
