"""Batched DHD prefill and decode on one GPU.

Mirrors reference pkg/src/kvlab/engine.py (ReuseSession :47-171,
prefill_with_selection :217-243, run_generation :298-328) and the reuse
forward of model.py:163-227, re-shaped for the B200:

prefill_batch(requests)                       one scheduled batch, all on device
  R2   kvs_pool_lookup            hit maps for every request at once
  G1   kvs_gather_kv              cached K/V rows (+RoPE re-alignment) into
                                  each request's arena pages, all layers
  probe fresh layer 0 over all rows (cuBLAS GEMMs + A1 on a scratch arena),
       layer-1 QKV: q dense, k_true into the arena for non-reused rows,
       v_true dense                                   (engine.py:182-207)
  D1   kvs_dhd_alpha              attention mass per key (tcgen05 2-pass)
  D2   kvs_dhd_select             dv-L1 x alpha, per-request radix top-B
  rows kvs_build_rows             S = non-reused U selected U {n-1}
  A1   layers 0..L-1 over rows S only: GEMM -> kvs_qkv_rope_scatter ->
       kvs_attention_fwd (tcgen05) -> GEMM(+residual)

decode_step(state, tokens)                    (engine.py:298-328, batched)
  probe query of the new tokens (layer 0 + layer-1 q), D3
  kvs_dhd_decode_select, then one layer-batched pass over chosen U {new}
  rows with kvs_decode_attention.

Only the projections are library GEMMs (torch.matmul -> cuBLAS); everything
else is libkvshare.so.  The residual stream is fp32, GEMM operands bf16.
"""
from __future__ import annotations

import os

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from .errors import InputError, ParameterError
from .model import HEAD_DIM, ToyModel
from .pool import PAGE_SIZE, CachePool, KVArena

TILE = 128


def h2d(a: np.ndarray, device) -> torch.Tensor:
    """Host array -> device without a stream sync: staged through the pinned
    caching host allocator (a pageable cudaMemcpyAsync waits for the stream)."""
    return torch.from_numpy(np.ascontiguousarray(a)).pin_memory().to(device, non_blocking=True)


class _Scratch:
    """Grow-only named device buffers for per-pass intermediates (residual
    stream, bf16 GEMM operand, QKV, Q, O).  Reuse is stream-ordered, like the
    caching allocator's, but sizes never churn, so the hot loop never reaches
    cudaMalloc."""

    def __init__(self, device):
        self.device = device
        self.bufs: dict = {}

    def get(self, name: str, shape, dtype) -> torch.Tensor:
        numel = int(np.prod(shape))
        b = self.bufs.get((name, dtype))
        if b is None or b.numel() < numel:
            # 25% headroom: a batch slightly larger than the last does not reallocate
            b = torch.empty(max(numel + numel // 4, 1), dtype=dtype, device=self.device)
            self.bufs[(name, dtype)] = b
        return b[:numel].view(*shape)


def budget(ratio: float, n_reused: int) -> int:
    """selection.py:51-52 with the reference's IEEE-double ceil."""
    return min(math.ceil(ratio * n_reused), n_reused)


@dataclass
class RowSet:
    """Query rows of a forward pass (grouped by request, ascending position)."""

    n_rows: int
    row_tok: torch.Tensor      # int32 flat token index
    row_req: torch.Tensor      # int32
    row_pos: torch.Tensor      # int32
    write_kv: torch.Tensor | None
    row_off: np.ndarray        # host [R+1]
    tiles: torch.Tensor | None = None   # int32 [3, n_tiles]
    n_tiles: int = 0

    def build_tiles(self, device, kv_len=None, partial_first: bool = False):
        """128-row query tiles, ordered longest-first (LPT) so the CTAs with
        the most keys start in the first wave and short tiles fill the tail.

        partial_first puts each request's ragged remainder tile at the FRONT
        (lowest positions, fewest keys) instead of the back (the tile that
        sees the whole context); only for row sets that are not the probe's
        aligned key tiles (D1's column-sum pass needs 128-aligned tiles).
        kv_len (per request, host) estimates a tile's key count when rows are
        a scattered subset; without it the cost is the row index itself."""
        off = np.asarray(self.row_off, dtype=np.int64)
        cnt = np.diff(off)
        ntile = (cnt + TILE - 1) // TILE
        req = np.repeat(np.arange(len(cnt), dtype=np.int64), ntile)
        first = np.repeat(np.cumsum(ntile) - ntile, ntile)
        k = np.arange(int(ntile.sum()), dtype=np.int64) - first
        if partial_first:
            rem = cnt[req] - (ntile[req] - 1) * TILE            # rows of the remainder tile
            row0 = off[req] + np.where(k == 0, 0, rem + (k - 1) * TILE)
            rows = np.where(k == 0, rem, TILE)
        else:
            row0 = off[req] + k * TILE
            rows = np.minimum(TILE, off[req + 1] - row0)
        self.n_tiles = int(ntile.sum())
        if self.n_tiles:
            last = row0 + rows - off[req]                          # rows up to the tile's end
            est = last.astype(np.float64)
            if kv_len is not None:
                est = est / np.maximum(cnt[req], 1) * np.asarray(kv_len, np.float64)[req]
            if os.environ.get("KVS_TILE_ORDER", "req") == "lpt":
                order = np.argsort(-est, kind="stable")
            else:
                # request-major, longest first within a request: the CTAs in
                # flight share one or two requests' K/V, which then stay in L2
                # (global LPT interleaved all requests and re-read K/V from
                # DRAM about 3x)
                order = np.lexsort((-est, req))
            t = np.stack([req[order], row0[order], rows[order]]).astype(np.int32)
        else:
            t = np.zeros((3, 1), dtype=np.int32)
        self.tiles = h2d(t, device)
        return self


@dataclass
class BatchState:
    """Device state of a batch of sequences (prefill and decode)."""

    lengths: np.ndarray                 # prefill lengths
    req_off_host: np.ndarray
    req_off: torch.Tensor               # int64 [R+1]
    tokens: torch.Tensor                # int64 flat prefill tokens
    pages: list                         # per request page lists
    block_table: torch.Tensor           # int32 [R, max_pages]
    batch_c: N.Batch
    capacity: np.ndarray                # token capacity per request
    src_slot: torch.Tensor | None = None
    src_cand: torch.Tensor | None = None
    n_hit_dev: torch.Tensor | None = None    # int32 [R] hit counts (device)
    selected: torch.Tensor | None = None   # uint8 flat
    dv_l1: torch.Tensor | None = None      # f32 flat (probe-layer deviation)
    alpha: torch.Tensor | None = None
    score: torch.Tensor | None = None
    eligible: torch.Tensor | None = None   # uint8 flat (decode-stage)
    rows: RowSet | None = None
    hidden_last: torch.Tensor | None = None  # fp32 [R, d_model]
    ctx_len: np.ndarray | None = None
    tokens_host: list = field(default_factory=list)
    budgets_dev: torch.Tensor | None = None

    def __del__(self):
        # pages not released, written back or handed on (st.pages = []) return
        # to the arena when the state goes away (reference sessions own numpy
        # caches that the GC frees; ours live in the shared arena)
        arena = getattr(self, "_arena", None)
        if arena is not None and self.pages:
            try:
                for p in self.pages:
                    arena.release(p)
            except Exception:                       # interpreter shutdown
                pass
            self.pages = []

    @property
    def n_hit(self) -> np.ndarray:
        """Host copy of the hit counts (synchronises; not used on the hot path)."""
        if self.n_hit_dev is None:
            return np.zeros(len(self.lengths), dtype=np.int64)
        return self.n_hit_dev.cpu().numpy().astype(np.int64)

    @n_hit.setter
    def n_hit(self, value):
        self.n_hit_dev = torch.as_tensor(np.asarray(value, dtype=np.int32)).to(self.req_off.device)

    @property
    def budgets(self):
        return None if self.budgets_dev is None else self.budgets_dev.cpu().numpy()


class _ProbeArena:
    """Scratch one-layer arena for the fresh layer-0 probe (all rows fresh)."""

    def __init__(self):
        self.data = None

    def get(self, cfg, n_pages, device):
        shape = (n_pages, 1, 2, PAGE_SIZE, cfg.kv_heads, HEAD_DIM)
        if self.data is None or self.data.shape[0] < n_pages or self.data.shape[1:] != shape[1:]:
            self.data = torch.zeros(shape, dtype=torch.bfloat16, device=device)
        return N.KVArena(self.data.data_ptr(), self.data.shape[0], 1, cfg.kv_heads, HEAD_DIM,
                         PAGE_SIZE)


class Engine:
    """Single-GPU executor of the KVShare hot path."""

    def __init__(self, model: ToyModel, pool: CachePool):
        self.model = model
        self.pool = pool
        self.cfg = model.config
        self.device = model.device
        self.arena: KVArena = pool.arena
        self.scale = 1.0 / math.sqrt(self.cfg.d_k)
        self._ws = {k: N.Workspace() for k in ("alpha", "select", "decode", "dsel")}
        self._probe_arena = _ProbeArena()
        # P1 decode-size projections, off by default: measured no faster than the library
        # GEMM at the decode step's 32 rows (profiles/r2_p1_skinny.txt)
        self.skinny = os.environ.get("KVS_SKINNY_PROJ", "0") != "0"
        self._wt = None
        self.rope_c = None
        if model.rope is not None:
            self.rope_c = N.Rope(model.rope[0].data_ptr(), model.rope[1].data_ptr(),
                                 self.cfg.max_positions)
        self.probe_layer = 1 if self.cfg.num_layers >= 2 else 0
        self.timers = None          # {name: [(start_event, end_event), ...]} when profiling
        self.fetcher = None         # shard.RemoteFetcher when the pool is sharded over GPUs
        self.peers = None           # shard.PeerArenas: remote shards read through peer memory
        self._events: list = []
        self._ev_next = 0
        self.scratch = _Scratch(self.device)
        self._xb_of = None
        # KVS_FUSED_Q_ROPE=1: A1 takes q straight from the projection rows and
        # rotates it in shared memory (the scatter then moves only k|v).  Off by
        # default: measured in the step, the rotation on the softmax warps' item
        # boundary costs more A1 time (+2.8 ms) than the scatter saves (-2.3 ms)
        self.fused_q_rope = os.environ.get("KVS_FUSED_Q_ROPE", "0") == "1"
        self.layer0_fast = True     # prefill_batch: probe layer 0 doubles as the prefill's
        self._side = torch.cuda.Stream(self.device) if torch.cuda.is_available() else None
        self._fetch_stream = torch.cuda.Stream(self.device) if torch.cuda.is_available() else None

    # ------------------------------------------------------------------ helpers
    def reset_timer_events(self, reserve: int = 0):
        """Reuse pre-created events (creating events inside a timed loop costs)."""
        while len(self._events) < reserve:
            self._events.append(torch.cuda.Event(enable_timing=True))
        self._ev_next = 0

    def _event(self):
        if self._ev_next == len(self._events):
            self._events.append(torch.cuda.Event(enable_timing=True))
        ev = self._events[self._ev_next]
        self._ev_next += 1
        return ev

    def _timed(self, name, fn, *args):
        if self.timers is None:
            return fn(*args)
        s, e = self._event(), self._event()
        s.record()
        out = fn(*args)
        e.record()
        self.timers.setdefault(name, []).append((s, e))
        return out

    def _rope(self):
        return self.rope_c

    def new_batch(self, token_lists, decode_capacity: int = 0,
                  tokens_dev: torch.Tensor | None = None) -> BatchState:
        lens = np.array([len(t) for t in token_lists], dtype=np.int64)
        if (lens <= 0).any():
            raise InputError("token sequence must be a non-empty 1-D array")
        off = np.zeros(len(lens) + 1, dtype=np.int64)
        off[1:] = np.cumsum(lens)
        if lens.max() + decode_capacity > self.cfg.max_positions:
            raise InputError("sequence longer than max_positions")
        dev = self.device
        if tokens_dev is None:
            flat = np.concatenate([np.asarray(t, dtype=np.int64) for t in token_lists])
            for t in token_lists:
                self.model.check_tokens(np.asarray(t, dtype=np.int64))
            tokens_dev = h2d(flat, dev)
        cap = lens + decode_capacity
        pages = [self.arena.alloc(self.arena.pages_for(int(c))) for c in cap]
        maxp = max(len(p) for p in pages)
        bt = np.zeros((len(lens), maxp), dtype=np.int32)
        for r, p in enumerate(pages):
            bt[r, :len(p)] = p
        req_off = h2d(off, dev)
        block_table = h2d(bt, dev)
        bc = N.Batch(len(lens), int(off[-1]), req_off.data_ptr(), block_table.data_ptr(), maxp)
        st = BatchState(lens, off, req_off, tokens_dev, pages, block_table, bc, cap)
        st.ctx_len = lens.copy()
        st._keep = (req_off, block_table)
        st._arena = self.arena
        return st

    def release(self, st: BatchState) -> None:
        for p in st.pages:
            self.arena.release(p)
        st.pages = []

    def _rows_all(self, st: BatchState) -> RowSet:
        """Every position of every request (probe / full recompute)."""
        dev = self.device
        n = int(st.req_off_host[-1])
        req = np.repeat(np.arange(len(st.lengths), dtype=np.int32), st.lengths)
        pos = np.concatenate([np.arange(l, dtype=np.int32) for l in st.lengths])
        rs = RowSet(n, torch.arange(n, dtype=torch.int32, device=dev),
                    h2d(req, dev), h2d(pos, dev), None,
                    st.req_off_host.copy())
        return rs.build_tiles(dev)

    def _attention(self, q, rows: RowSet, layer: int, arena_c, batch_c, out, lse=None):
        self._timed("attention", N.call, "kvs_attention_fwd", q.data_ptr(), rows.row_pos.data_ptr(), rows.n_rows,
               self.cfg.num_heads, rows.tiles[0].data_ptr(), rows.tiles[1].data_ptr(),
               rows.tiles[2].data_ptr(), rows.n_tiles, None, 1, layer, arena_c, batch_c,
               self.scale, N.ptr(out), N.ptr(lse), N.stream_ptr())
        g = self.cfg.num_heads // self.cfg.kv_heads
        if g % 2 == 1 and g > 1 and out is not None and rows.n_tiles > 0:
            N.launch_count["kernels"] += 1      # odd groups: head-pair + single-head launches

    def _attention_qkv(self, qkv, rows: RowSet, layer: int, arena_c, batch_c, out):
        """A1 reading the un-rotated query heads straight from the QKV
        projection rows (rotated in the kernel's shared memory): the scatter
        then moves only k|v (no q round trip through HBM)."""
        self._timed("attention", N.call, "kvs_attention_fwd_qkv", qkv.data_ptr(), qkv.shape[1],
                    self._rope(), rows.row_pos.data_ptr(), rows.n_rows, self.cfg.num_heads,
                    rows.tiles[0].data_ptr(), rows.tiles[1].data_ptr(), rows.tiles[2].data_ptr(),
                    rows.n_tiles, None, 1, layer, arena_c, batch_c, self.scale, out.data_ptr(),
                    N.stream_ptr())

    def _decode_attention(self, q, rows: RowSet, layer: int, arena_c, batch_c, out, max_kv):
        cfg = self.cfg
        nb = N.ws_bytes("kvs_decode_attention_workspace", rows.n_rows, cfg.num_heads,
                        cfg.kv_heads, HEAD_DIM, max_kv)
        ws = self._ws["decode"].get(nb, self.device)
        N.call("kvs_decode_attention", q.data_ptr(), rows.row_req.data_ptr(),
               rows.row_pos.data_ptr(), rows.n_rows, cfg.num_heads, None, 1, layer, arena_c,
               batch_c, self.scale, out.data_ptr(), ws.data_ptr(), ws.numel(), N.stream_ptr())

    def _scatter(self, qkv, rows: RowSet, layer, arena_c, batch_c, q_out, write_kv=None,
                 k_out=None, v_out=None, use_write=True, src_row=None):
        wk = write_kv if write_kv is not None else (rows.write_kv if use_write else None)
        if src_row is not None:
            N.call("kvs_qkv_rope_scatter_rows", qkv.data_ptr(), src_row.data_ptr(), rows.n_rows,
                   self.cfg.num_heads, rows.row_req.data_ptr(), rows.row_pos.data_ptr(),
                   N.ptr(wk), layer, arena_c, batch_c, self._rope(), N.ptr(q_out),
                   N.ptr(k_out), N.ptr(v_out), N.stream_ptr())
            return
        N.call("kvs_qkv_rope_scatter", qkv.data_ptr(), rows.n_rows, self.cfg.num_heads,
               rows.row_req.data_ptr(), rows.row_pos.data_ptr(), N.ptr(wk), layer, arena_c,
               batch_c, self._rope(), N.ptr(q_out), N.ptr(k_out), N.ptr(v_out),
               N.stream_ptr())

    def _embed(self, tokens_flat, rows: RowSet, scratch: bool = False) -> torch.Tensor:
        """fp32 residual stream of the rows.  scratch=True places it in the
        engine's reusable buffer (the caller consumes it within the pass)."""
        n, d = rows.n_rows, self.cfg.d_model
        xb = self.scratch.get("xb", (n, d), torch.bfloat16)
        x = self.scratch.get("x", (n, d), torch.float32) if scratch else \
            torch.empty(n, d, dtype=torch.float32, device=self.device)
        N.call("kvs_embed_rows", self.model.embedding.data_ptr(), d,
               tokens_flat.data_ptr(), rows.row_tok.data_ptr(), n, xb.data_ptr(),
               x.data_ptr(), N.stream_ptr())
        self._xb_of = (x.data_ptr(), n)     # xb == bf16(x) until x changes
        return x

    def forward_rows(self, x, rows: RowSet, layers, arena_c, batch_c, decode=False,
                     max_kv=0, write_kv_per_layer=None, capture=None, first_qkv=None):
        """Layer loop over a row set: x (fp32 [n, d_model]) updated in place.
        first_qkv = (qkv, src_row): the first layer's projection rows already
        exist (row i is qkv[src_row[i]]) and are not recomputed."""
        cfg, m = self.cfg, self.model
        H, n = cfg.num_heads, rows.n_rows
        q = self.scratch.get("q", (n, H, HEAD_DIM), torch.bfloat16)
        o = self.scratch.get("o", (n, H, HEAD_DIM), torch.bfloat16)
        for i, layer in enumerate(layers):
            wk = write_kv_per_layer[layer] if write_kv_per_layer is not None else None
            if i == 0 and first_qkv is not None:
                self._scatter(first_qkv[0], rows, layer, arena_c, batch_c, q, write_kv=wk,
                              src_row=first_qkv[1])
            elif not decode and capture is None and self.fused_q_rope:
                # q stays in the projection rows; A1 rotates it in shared memory
                qkv = self._qkv(x, layer)
                self._scatter(qkv, rows, layer, arena_c, batch_c, None, write_kv=wk)
                self._attention_qkv(qkv, rows, layer, arena_c, batch_c, o)
                self._out_proj(x, o, layer)
                continue
            else:
                qkv = self._qkv(x, layer)
                self._scatter(qkv, rows, layer, arena_c, batch_c, q, write_kv=wk)
            if decode:
                self._decode_attention(q, rows, layer, arena_c, batch_c, o, max_kv)
            else:
                self._attention(q, rows, layer, arena_c, batch_c, o)
            if capture is not None:
                capture.append((layer, q.clone(), o.clone()))
            self._out_proj(x, o, layer)
            if capture is not None:
                capture.append((layer, "hidden", x.clone()))
        return x

    SKINNY_MAX_ROWS = 64

    def _skinny_ok(self, n: int) -> bool:
        """Decode-size row counts take P1 (kvs_proj_skinny) when the widths allow."""
        cfg = self.cfg
        return (self.skinny and 1 <= n <= self.SKINNY_MAX_ROWS and cfg.d_model % 512 == 0
                and (cfg.num_heads * HEAD_DIM) % 512 == 0 and cfg.d_model % 128 == 0
                and self.model.w_qkv[0].shape[1] % 128 == 0)

    @staticmethod
    def pack_skinny(w: torch.Tensor) -> torch.Tensor:
        """W [k][n] -> P1's layout: 16 x 64 tiles of W^T, [n/16][k/64][16][64]
        (include/kvshare.h, kvs_proj_skinny)."""
        k, n = w.shape
        return w.t().reshape(n // 16, 16, k // 64, 64).permute(0, 2, 1, 3).contiguous()

    def ensure_skinny_weights(self) -> None:
        """P1-packed copies of every layer's projection weights.  Built once,
        outside any graph capture."""
        if self._wt is not None or not self._skinny_ok(1):
            return
        m = self.model
        self._wt = ([self.pack_skinny(w) for w in m.w_qkv], [self.pack_skinny(w) for w in m.w_o])

    def _qkv(self, x: torch.Tensor, layer: int) -> torch.Tensor:
        """bf16(x) @ W_qkv into scratch (model.py:193-195)."""
        n = x.shape[0]
        w = self.model.w_qkv[layer]
        xb = self.scratch.get("xb", (n, x.shape[1]), torch.bfloat16)
        if self._xb_of != (x.data_ptr(), n):
            xb.copy_(x)
            self._xb_of = (x.data_ptr(), n)
        qkv = self.scratch.get("qkv", (n, w.shape[1]), torch.bfloat16)
        if self._skinny_ok(n):
            self.ensure_skinny_weights()
            N.call("kvs_proj_skinny", xb.data_ptr(), n, self._wt[0][layer].data_ptr(),
                   w.shape[1], w.shape[0], 0, qkv.data_ptr(), None, N.stream_ptr())
            return qkv
        return torch.matmul(xb, w, out=qkv)

    def _out_proj(self, x: torch.Tensor, o: torch.Tensor, layer: int) -> None:
        """x += merge(o) @ W_o in place (model.py:202): the residual add runs in
        the cuBLAS epilogue with C = D = x (fp32), A/B bf16 - no copy of x.
        Decode-size row counts run P1, whose epilogue also leaves bf16(x) in
        the next projection's operand buffer."""
        n = x.shape[0]
        if self._skinny_ok(n):
            self.ensure_skinny_weights()
            xb = self.scratch.get("xb", (n, x.shape[1]), torch.bfloat16)
            N.call("kvs_proj_skinny", o.data_ptr(), n, self._wt[1][layer].data_ptr(),
                   x.shape[1], o[0].numel(), 1, x.data_ptr(), xb.data_ptr(), N.stream_ptr())
            self._xb_of = (x.data_ptr(), n)
            return
        torch.addmm(x, o.view(n, -1), self.model.w_o[layer], out_dtype=torch.float32, out=x)
        self._xb_of = None

    # ------------------------------------------------------------------ prefill
    def lookup(self, st: BatchState):
        """R2 for the whole batch; hit counts stay on the device (no sync)."""
        res = self.pool.lookup_device(st.tokens, st.req_off, st.req_off_host)
        st.src_slot, st.src_cand = res.src_slot, res.src_cand
        st.n_hit_dev = res.n_hit
        st._contributed = res.contributed
        return st

    def set_hits(self, st: BatchState, hits) -> None:
        """Hit maps from CachePool.admit for the batch's requests, in order."""
        if len(hits) != len(st.lengths) or any(h.length != int(l) for h, l in zip(hits, st.lengths)):
            raise InputError("admitted hit maps do not match the batch's requests")
        st.src_slot = torch.cat([h.src_slot for h in hits])
        st.src_cand = torch.cat([h.src_cand for h in hits])
        st.n_hit = np.array([h.n_hit for h in hits], dtype=np.int64)

    def gather(self, st: BatchState, layers=None, slot=None, remote: bool = True):
        """G1 for layers [begin, end) (all by default); `slot` overrides the
        hit map (e.g. with selected rows masked out).  remote=False leaves the
        rows of other GPUs' shards to the caller."""
        if not self.pool.entries and not self.pool._retired:
            return
        begin, end = layers if layers is not None else (0, self.cfg.num_layers)
        idx = self.pool._build_index()
        slot = st.src_slot if slot is None else slot
        if self.peers is not None:
            # remote shards' rows read from their owners' arenas in the same launch
            self._timed("gather", self.peers.gather, st, idx, slot, (begin, end))
            return
        if self.fetcher is not None:
            # remote-shard rows come through the fetcher (plain path: whole
            # exchange here; the fast path of prefill_batch overlaps it)
            slot = self.fetcher.local_mask(slot, idx)
            if remote:
                self._timed("remote_fetch", self.fetcher.fetch, st, idx, (begin, end))
        self._timed("gather", N.call, "kvs_gather_kv", self.arena.c, st.batch_c, slot.data_ptr(),
               st.src_cand.data_ptr(), idx["slot_pages"].data_ptr(), idx["slot_max_pages"], begin,
               end, self._rope(), N.stream_ptr())

    def _probe(self, st: BatchState, write_k: bool = True, layer0_in_place: bool = False,
               k_out: torch.Tensor | None = None):
        """engine.py:182-207: fresh layers below the probe over ALL rows, then
        the probe layer's q (dense), k_true (into the arena for non-reused
        rows, so the arena layer holds k_pert) and v_true (dense).

        Layer 0 runs on a scratch arena, or - layer0_in_place - on the
        request's own layer-0 pages (fresh K/V for every row; the caller
        gathers the cached rows back afterwards for the reused, unselected
        positions).  In place, the layer-0 hidden rows are kept on the state
        (st._x_probe): layer 0's K/V are context-free, so they equal the
        partial prefill's layer 0 (reference test_model.py:121-128)."""
        cfg, m, dev = self.cfg, self.model, self.device
        H, G = cfg.num_heads, cfg.kv_heads
        rows = self._rows_all(st)
        n = rows.n_rows
        x = self._embed(st.tokens, rows, scratch=True)
        p = self.probe_layer
        if p == 1 and layer0_in_place:
            q = self.scratch.get("q", (n, H, HEAD_DIM), torch.bfloat16)
            o = self.scratch.get("o", (n, H, HEAD_DIM), torch.bfloat16)
            qkv = self._qkv(x, 0)
            if self.fused_q_rope:
                self._scatter(qkv, rows, 0, self.arena.c, st.batch_c, None, use_write=False)
                self._attention_qkv(qkv, rows, 0, self.arena.c, st.batch_c, o)
            else:
                self._scatter(qkv, rows, 0, self.arena.c, st.batch_c, q, use_write=False)
                self._attention(q, rows, 0, self.arena.c, st.batch_c, o)
            self._out_proj(x, o, 0)
            st._x_probe = x
        elif p == 1:
            npages = int(sum((l + PAGE_SIZE - 1) // PAGE_SIZE for l in st.lengths))
            parena = self._probe_arena.get(cfg, npages, dev)
            bt = np.zeros((len(st.lengths), st.block_table.shape[1]), dtype=np.int32)
            base = 0
            for r, l in enumerate(st.lengths):
                k = (l + PAGE_SIZE - 1) // PAGE_SIZE
                bt[r, :k] = np.arange(base, base + k)
                base += k
            pbt = h2d(bt, dev)
            pbatch = N.Batch(st.batch_c.n_req, st.batch_c.n_total, st.req_off.data_ptr(),
                             pbt.data_ptr(), bt.shape[1])
            q = self.scratch.get("q", (n, H, HEAD_DIM), torch.bfloat16)
            o = self.scratch.get("o", (n, H, HEAD_DIM), torch.bfloat16)
            qkv = self._qkv(x, 0)
            self._scatter(qkv, rows, 0, parena, pbatch, q, use_write=False)
            self._attention(q, rows, 0, parena, pbatch, o)
            self._out_proj(x, o, 0)
            st._probe_keep = pbt
        qkv = self._qkv(x, p)
        q1 = torch.empty(n, H, HEAD_DIM, dtype=torch.bfloat16, device=dev)
        v_true = torch.empty(n, G, HEAD_DIM, dtype=torch.bfloat16, device=dev)
        wk = (st.src_slot < 0).to(torch.uint8) if write_k else \
            torch.zeros(n, dtype=torch.uint8, device=dev)
        self._scatter(qkv, rows, p, self.arena.c, st.batch_c, q1, write_kv=wk, k_out=k_out,
                      v_out=v_true)
        if p == 1 and layer0_in_place:
            # rows S of this all-row layer-1 projection are the partial
            # prefill's layer-1 projection (same x rows): session_forward reuses
            # them; the buffer stays intact until its layer-2 GEMM
            st._qkv1 = qkv
        return rows, q1, v_true

    def _select(self, st: BatchState, v_true, alpha, budgets):
        dev, n = self.device, int(st.req_off_host[-1])
        bud = budgets if torch.is_tensor(budgets) else \
            h2d(np.asarray(budgets, dtype=np.int32), dev)
        dv = torch.empty(n, dtype=torch.float32, device=dev)
        score = torch.empty(n, dtype=torch.float32, device=dev)
        sel = torch.empty(n, dtype=torch.uint8, device=dev)
        ws = self._ws["select"].get(N.ws_bytes("kvs_dhd_select_workspace", n, len(st.lengths)),
                                    dev, zero=True)
        self._timed("dhd_select", N.call, "kvs_dhd_select", v_true.data_ptr(), alpha.data_ptr(),
                    st.src_slot.data_ptr(), self.probe_layer, self.arena.c, st.batch_c,
                    bud.data_ptr(), dv.data_ptr(), score.data_ptr(), sel.data_ptr(),
                    ws.data_ptr(), ws.numel(), N.stream_ptr())
        st._bud = bud
        return dv, score, sel

    def probe_and_select(self, st: BatchState, ratio: float, layer0_in_place: bool = False):
        """engine.py:233-243 (PRACTICAL): fresh probe, D1 alpha, D2 select."""
        cfg, dev = self.cfg, self.device
        H, G = cfg.num_heads, cfg.kv_heads
        rows, q1, v_true = self._probe(st, layer0_in_place=layer0_in_place)
        n = rows.n_rows
        alpha = torch.empty(n, dtype=torch.float32, device=dev)
        ws = self._ws["alpha"].get(N.ws_bytes("kvs_dhd_alpha_workspace", n, H, G), dev)
        if getattr(st, "_before_alpha", None) is not None:
            st._before_alpha()                                     # remote rows (sharded pool)
            st._before_alpha = None
        if getattr(st, "_gathered", None) is not None:
            torch.cuda.current_stream().wait_event(st._gathered)     # k_pert complete
            st._gathered = None
        self._timed("dhd_alpha", N.call, "kvs_dhd_alpha", q1.data_ptr(), H, 1, self.probe_layer, self.arena.c, st.batch_c,
               rows.row_pos.data_ptr(), rows.tiles[0].data_ptr(), rows.tiles[1].data_ptr(),
               rows.tiles[2].data_ptr(), rows.n_tiles, None, self.scale, alpha.data_ptr(),
               ws.data_ptr(), ws.numel(), N.stream_ptr())
        if getattr(st, "n_hit_dev", None) is not None:
            # selection.py:51-52 on the device: IEEE-double product, ceil, clamp
            nh = st.n_hit_dev.to(torch.float64)
            bud = torch.minimum(torch.ceil(nh * float(ratio)), nh).to(torch.int32)
        else:
            bud = torch.from_numpy(np.array([budget(ratio, int(h)) for h in st.n_hit],
                                            dtype=np.int32)).to(self.device)
        st.budgets_dev = bud
        st.dv_l1, st.score, st.selected = self._select(st, v_true, alpha, bud)
        st.alpha = alpha
        st._probe_q, st._probe_v_true = q1, v_true
        return st

    def build_rows(self, st: BatchState, selected: torch.Tensor | None) -> RowSet:
        dev, R = self.device, len(st.lengths)
        counts = torch.empty(R, dtype=torch.int32, device=dev)
        src = st.src_slot if st.src_slot is not None else \
            torch.full((int(st.req_off_host[-1]),), -1, dtype=torch.int32, device=dev)
        N.call("kvs_build_rows", st.req_off.data_ptr(), R, src.data_ptr(), N.ptr(selected),
               counts.data_ptr(), None, None, None, None, None, N.stream_ptr())
        c = counts.cpu().numpy().astype(np.int64)                         # sync 2
        off = np.zeros(R + 1, dtype=np.int64)
        off[1:] = np.cumsum(c)
        n = int(off[-1])
        row_off = h2d(off, dev)
        rows = RowSet(n, torch.empty(n, dtype=torch.int32, device=dev),
                      torch.empty(n, dtype=torch.int32, device=dev),
                      torch.empty(n, dtype=torch.int32, device=dev),
                      torch.empty(n, dtype=torch.uint8, device=dev), off)
        N.call("kvs_build_rows", st.req_off.data_ptr(), R, src.data_ptr(), N.ptr(selected),
               None, row_off.data_ptr(), rows.row_tok.data_ptr(), rows.row_req.data_ptr(),
               rows.row_pos.data_ptr(), rows.write_kv.data_ptr(), N.stream_ptr())
        rows._keep = (row_off, src)
        return rows.build_tiles(dev, kv_len=st.lengths, partial_first=True)

    def session_forward(self, st: BatchState, rows: RowSet, capture=None, x_probe=None):
        """Layers over rows S.  With x_probe (the probe's all-row hidden state
        after layer 0) the pass starts at layer 1 from rows S of it."""
        if x_probe is not None:
            x = self.scratch.get("x_s", (rows.n_rows, self.cfg.d_model), torch.float32)
            torch.index_select(x_probe, 0, rows.row_tok, out=x)
            first = 1
        else:
            x = self._embed(st.tokens, rows, scratch=capture is None)
            first = 0
        st.session_first = first
        qkv1 = getattr(st, "_qkv1", None) if x_probe is not None else None
        st._qkv1 = None
        x = self.forward_rows(x, rows, range(first, self.cfg.num_layers), self.arena.c,
                              st.batch_c, capture=capture,
                              first_qkv=(qkv1, rows.row_tok) if qkv1 is not None else None)
        keep = getattr(rows, "_keep", None)
        # last row of each request: from the device copy of row_off when the
        # row set was built on the device (no host->device copy here)
        last = keep[0][1:] - 1 if keep is not None else h2d(rows.row_off[1:] - 1, self.device)
        st.rows = rows
        st.hidden_last = x[last]
        return x

    def prefill_batch(self, token_lists, ratio: float = 0.2, mode: str = "selective",
                      decode_capacity: int = 0, tokens_dev=None, hits=None) -> BatchState:
        """One scheduled batch through the hot path (modes: selective / naive / full).
        hits: the requests' admission-time hit maps (CachePool.admit results,
        simulate.py:180-186, 264-266) instead of a lookup at batch time."""
        if not 0.0 <= ratio <= 1.0:
            raise ParameterError(f"ratio must lie in [0, 1], got {ratio}")
        st = self.new_batch(token_lists, decode_capacity, tokens_dev)
        if hits is not None and mode != "full":
            self.set_hits(st, hits)
            if not int(st.n_hit.sum()):
                hits = None
                mode = "full"
        if mode == "full" or (hits is None and not self.pool.entries):
            st.n_hit_dev = torch.zeros(len(st.lengths), dtype=torch.int32, device=self.device)
            rows = self.build_rows(st, None)
            rows.write_kv.fill_(1)
            self.session_forward(st, rows)
            st.selected = None
            return st
        if hits is None:
            self.lookup(st)
        L = self.cfg.num_layers
        if mode == "selective" and ratio > 0 and self.probe_layer == 1 and self.layer0_fast:
            # layers >= 1 gathered first; the probe's fresh layer 0 runs in
            # place and doubles as the partial prefill's layer 0; cached layer-0
            # rows return for the reused, unselected positions after selection
            # G1 (HBM-bound) runs on a side stream under the probe's layer 0
            # (tensor-bound); D1 reads layer 1's k_pert, so it waits for it.
            # With a sharded pool the remote rows' exchange also runs off the
            # main stream: planned and counted right after the lookup, moved
            # and unpacked while the probe computes (st._before_alpha).
            main = torch.cuda.current_stream()
            self._side.wait_stream(main)
            rf = None
            if self.fetcher is not None:
                idx = self.pool._build_index()
                self._fetch_stream.wait_stream(main)
                with torch.cuda.stream(self._fetch_stream):
                    rf = self.fetcher.begin(st, idx)
            with torch.cuda.stream(self._side):
                self.gather(st, (1, L), remote=False)
                gathered = torch.cuda.Event()
                gathered.record()
            st._gathered = gathered
            if rf is not None:
                def before_alpha():
                    with torch.cuda.stream(self._fetch_stream):
                        self._timed("remote_fetch", rf.finish)
                        rf.unpack(st, (1, L))
                    main.wait_stream(self._fetch_stream)
                    for t in (rf.rows, rf.flat_t, rf.cand):          # layer 0 later on main
                        if t is not None:
                            t.record_stream(main)
                st._before_alpha = before_alpha
            self.probe_and_select(st, ratio, layer0_in_place=True)
            keep = torch.where(st.selected.bool(), torch.full_like(st.src_slot, -1), st.src_slot)
            self.gather(st, (0, 1), slot=keep, remote=False)
            if rf is not None:
                rf.unpack(st, (0, 1), skip=st.selected)
                st._remote_fetch = rf
            rows = self.build_rows(st, st.selected)
            self.session_forward(st, rows, x_probe=st._x_probe)
            st._x_probe = None
        else:
            self.gather(st)
            if mode == "selective" and ratio > 0:
                self.probe_and_select(st, ratio)
                rows = self.build_rows(st, st.selected)
            else:
                rows = self.build_rows(st, None)
                st.selected = None
            self.session_forward(st, rows)
        reused = st.src_slot >= 0
        sel = st.selected.bool() if st.selected is not None else torch.zeros_like(reused)
        st.eligible = (reused & ~sel).to(torch.uint8)
        return st

    def forward_all_rows(self, st: BatchState, write_kv: torch.Tensor, capture=None):
        """Every row of every request through every layer (model.py:163-208):
        K/V are written for rows with write_kv set (uint8, flat over the
        batch) and kept as gathered elsewhere - model_forward (all ones),
        model_forward_with_reuse / a PRACTICAL session's prefill (not reused
        or recomputed).  capture receives (layer, q, o) and (layer, "hidden",
        x) like forward_rows."""
        rows = self._rows_all(st)
        x = self._embed(st.tokens, rows)
        L = self.cfg.num_layers
        x = self.forward_rows(x, rows, range(L), self.arena.c, st.batch_c,
                              write_kv_per_layer=[write_kv] * L, capture=capture)
        st.rows = rows
        st.hidden_last = x[h2d(st.req_off_host[1:] - 1, self.device)]
        return x

    def refresh_lru(self, st: BatchState):
        c = st._contributed.cpu().numpy()
        for r in range(c.shape[0]):
            self.pool.refresh_lru(c[r])

    # ------------------------------------------------------------------ decode
    def ensure_dv(self, st: BatchState):
        """delta_v_probe support (engine.py:81-89, 140-148) for batches that did
        not run the DHD probe: v_true from a fresh probe (no arena writes),
        dv-L1 against the cached probe-layer V."""
        if st.dv_l1 is not None:
            return
        n = int(st.req_off_host[-1])
        if st.src_slot is None or not bool((st.src_slot >= 0).any()):
            st.dv_l1 = torch.zeros(n, dtype=torch.float32, device=self.device)
            return
        _, _, v_true = self._probe(st, write_k=False)
        zeros = torch.zeros(n, dtype=torch.float32, device=self.device)
        st.dv_l1, _, _ = self._select(st, v_true, zeros, np.zeros(len(st.lengths), np.int32))

    def probe_query(self, st: BatchState, new_tokens) -> torch.Tensor:
        """query_rows_probe (engine.py:150-171) for every request's next token:
        layers below the probe over cache + own row, then the probe-layer q.
        new_tokens: host array or device int64 tensor [R]."""
        cfg, dev = self.cfg, self.device
        R = len(st.lengths)
        pos = self._ctx_dev(st)
        rows = RowSet(R, torch.arange(R, dtype=torch.int32, device=dev),
                      torch.arange(R, dtype=torch.int32, device=dev), pos, None,
                      np.arange(R + 1, dtype=np.int64))
        tok = new_tokens if torch.is_tensor(new_tokens) else \
            h2d(np.asarray(new_tokens, dtype=np.int64), dev)
        x = self._embed(tok, rows)
        max_kv = int(st.capacity.max())
        x = self.forward_rows(x, rows, range(self.probe_layer), self.arena.c, st.batch_c,
                              decode=True, max_kv=max_kv)
        qkv = self._qkv(x, self.probe_layer)
        q = torch.empty(R, cfg.num_heads, HEAD_DIM, dtype=torch.bfloat16, device=dev)
        zero = torch.zeros(R, dtype=torch.uint8, device=dev)
        self._scatter(qkv, rows, self.probe_layer, self.arena.c, st.batch_c, q, write_kv=zero)
        return q

    def _ctx_dev(self, st: BatchState) -> torch.Tensor:
        """Device copy of the current context lengths (int32), refreshed when
        the host value changes (pinned H2D, no sync)."""
        key = getattr(st, "_ctx_key", None)
        cur = st.ctx_len.tobytes()
        if key != cur:
            st._ctx_dev = h2d(st.ctx_len.astype(np.int32), self.device)
            st._ctx_key = cur
        return st._ctx_dev

    def decode_select_device(self, st: BatchState, q_t: torch.Tensor, n_extra: int):
        """D3 (selection.py:80-105) for every request, on the device: returns
        (chosen [R, n_extra] int32 ascending, -1 padded; n_chosen [R]) and
        clears the chosen rows from st.eligible.  No host synchronisation."""
        cfg, dev, R = self.cfg, self.device, len(st.lengths)
        ctx = self._ctx_dev(st)
        # workspace and logits stride sized by the capacity, not the current
        # context: the same launch is valid at every step (CUDA-graph replay)
        max_ctx = int(st.capacity.max())
        chosen = torch.empty(R, max(n_extra, 1), dtype=torch.int32, device=dev)
        nch = torch.zeros(R, dtype=torch.int32, device=dev)
        ws = self._ws["dsel"].get(N.ws_bytes("kvs_dhd_decode_select_workspace", R, cfg.num_heads,
                                             max_ctx), dev, zero=True)
        self._timed("dhd_decode", N.call, "kvs_dhd_decode_select", q_t.data_ptr(), cfg.num_heads,
                    ctx.data_ptr(), max_ctx, st.dv_l1.data_ptr(), st.eligible.data_ptr(),
                    self.probe_layer, self.arena.c, st.batch_c, n_extra, self.scale,
                    chosen.data_ptr(), nch.data_ptr(), None, ws.data_ptr(), ws.numel(),
                    N.stream_ptr())
        return chosen, nch

    def decode_select(self, st: BatchState, q_t: torch.Tensor, n_extra: int):
        """decode_select_device with the choices as host lists (synchronises)."""
        chosen, nch = self.decode_select_device(st, q_t, n_extra)
        ch, nc = chosen.cpu().numpy(), nch.cpu().numpy()
        return [[int(x) for x in ch[r, :nc[r]]] for r in range(len(st.lengths))]

    def decode_step_device(self, st: BatchState, new_tokens: torch.Tensor, n_extra: int):
        """One decode token per request (engine.py:312-327) with no host
        round trip: probe query, D3, then the chosen rows and the new token as
        one layer-batched pass.  The pass has a fixed
        n_extra + 1 row slots per request; slots D3 left empty (-1) keep their
        K/V untouched and their outputs are discarded.  new_tokens: device
        int64 [R].  Returns (hidden of the new rows [R, d_model] fp32,
        chosen [R, n_extra] int32 -1 padded, n_chosen [R] int32)."""
        R, dev = len(st.lengths), self.device
        if (st.ctx_len + 1 > st.capacity).any():
            raise InputError("decode capacity exhausted")
        E = max(int(n_extra), 0)
        ctx = self._ctx_dev(st)
        if E > 0 and st.eligible is not None:
            self.ensure_dv(st)
            q_t = self.probe_query(st, new_tokens)
            chosen, nch = self.decode_select_device(st, q_t, E)
        else:
            chosen = torch.full((R, max(E, 1)), -1, dtype=torch.int32, device=dev)[:, :E]
            nch = torch.zeros(R, dtype=torch.int32, device=dev)
        pos = torch.cat([chosen, ctx[:, None]], dim=1)                    # [R, E + 1]
        valid = pos >= 0
        pos_c = pos.clamp(min=0)
        prev = st.req_off[:-1, None] + pos_c[:, :E].to(torch.int64)       # prefill rows only
        tok = torch.cat([st.tokens[prev.clamp(max=st.tokens.numel() - 1)],
                         new_tokens.view(R, 1).to(torch.int64)], dim=1).reshape(-1)
        n = R * (E + 1)
        rows = RowSet(n, torch.arange(n, dtype=torch.int32, device=dev),
                      torch.arange(R, dtype=torch.int32, device=dev).repeat_interleave(E + 1),
                      pos_c.reshape(-1).to(torch.int32), valid.reshape(-1).to(torch.uint8),
                      np.arange(0, n + 1, E + 1, dtype=np.int64))
        x = self._embed(tok, rows)
        x = self.forward_rows(x, rows, range(self.cfg.num_layers), self.arena.c, st.batch_c,
                              decode=True, max_kv=int(st.capacity.max()))
        ctx.add_(1)                        # the device context counter moves with the host one
        self._advance_ctx_host(st, new_tokens)
        return x.view(R, E + 1, -1)[:, E], chosen, nch

    @staticmethod
    def _advance_ctx_host(st: BatchState, new_tokens) -> None:
        st.ctx_len = st.ctx_len + 1
        st._ctx_key = st.ctx_len.tobytes()
        st._decoded = getattr(st, "_decoded", []) + [new_tokens]

    def decode_graph(self, st: BatchState, n_extra: int) -> "DecodeGraph":
        """decode_step_device captured once as a CUDA graph for this batch
        (about 140 launches per token step replayed without host work)."""
        return DecodeGraph(self, st, n_extra)

    def decode_step(self, st: BatchState, new_tokens, n_extra: int):
        """decode_step_device for host tokens, choices returned as host lists
        (one synchronisation, for the reference-shaped API)."""
        R = len(st.lengths)
        tok = h2d(np.asarray(new_tokens, dtype=np.int64).reshape(R), self.device)
        h, chosen, nch = self.decode_step_device(st, tok, n_extra)
        ch, nc = chosen.cpu().numpy(), nch.cpu().numpy()
        return h, [[int(x) for x in ch[r, :nc[r]]] for r in range(R)]

    # ------------------------------------------------------------------ write-back
    def write_back(self, st: BatchState, request_ids) -> None:
        """Finished requests become pool entries (zero-copy; simulate.py:207-210)."""
        flat = None
        for r, rid in enumerate(request_ids):
            if flat is None:
                flat = st.tokens.cpu().numpy()
            toks = flat[st.req_off_host[r]:st.req_off_host[r + 1]]
            self.pool.insert_pages(rid, toks, st.pages[r])
        st.pages = []


class DecodeGraph:
    """One decode token step of a batch (Engine.decode_step_device: probe
    query, D3, chosen U {new} rows through every layer) as a CUDA graph.

    The step's launches only depend on the batch's device state (block
    table, eligibility, dv-L1, the device context counter it advances itself)
    and on static shapes, so it is captured once and replayed per token: the
    host issues one graph launch instead of ~140 kernel launches and the
    Python around them.  The graph owns its scratch and workspace buffers
    (the engine's grow-only buffers may be reallocated by later work).
    replay(new_tokens) returns the same (hidden, chosen, n_chosen) tensors
    every step - static outputs, overwritten by the next replay."""

    def __init__(self, eng: Engine, st: BatchState, n_extra: int):
        """Capture after at least one eager decode step of this batch (it
        initialises cuBLAS for the step's shapes)."""
        self.eng, self.st, self.n_extra = eng, st, int(n_extra)
        R, dev = len(st.lengths), eng.device
        if self.n_extra > 0 and st.eligible is not None:
            eng.ensure_dv(st)                       # host-dependent set-up stays outside
        eng._ctx_dev(st)
        eng.ensure_skinny_weights()
        self.tok = torch.zeros(R, dtype=torch.int64, device=dev)
        saved = (eng.scratch, eng._ws, eng.timers)
        # the graph's own buffers, allocated while capturing (from the graph's
        # private memory pool), sized for this step only
        self.scratch = _Scratch(dev)
        self.ws = {k: N.Workspace() for k in saved[1]}
        ctx_host, key, dec = st.ctx_len.copy(), getattr(st, "_ctx_key", None), \
            list(getattr(st, "_decoded", []))
        eng.scratch, eng._ws, eng.timers, eng._xb_of = self.scratch, self.ws, None, None
        try:
            torch.cuda.synchronize()
            # capture records the launches without running them; the host-side
            # context bookkeeping the captured call did is undone
            self.graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.graph):
                self.out = eng.decode_step_device(st, self.tok, self.n_extra)
            st.ctx_len, st._ctx_key, st._decoded = ctx_host, key, dec
        finally:
            eng.scratch, eng._ws, eng.timers = saved
            eng._xb_of = None

    def replay(self, new_tokens: torch.Tensor):
        st = self.st
        if (st.ctx_len + 1 > st.capacity).any():
            raise InputError("decode capacity exhausted")
        self.tok.copy_(new_tokens.view(-1), non_blocking=True)
        self.graph.replay()
        Engine._advance_ctx_host(st, new_tokens)
        return self.out

