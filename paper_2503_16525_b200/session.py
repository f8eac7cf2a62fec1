"""Reference-shaped sessions, forwards and generation over the device engine.

Drop-ins for reference pkg/src/kvlab/model.py (``LayerStates`` :132-151,
``model_forward`` :211-213, ``model_forward_with_reuse`` :216-227) and
pkg/src/kvlab/engine.py (``ReuseSession`` :47-171, ``PrefillResult`` :174-179,
``prefill_with_selection`` :217-243, ``GenerationResult`` :288-295,
``run_generation`` :298-328).  Each call runs the batched engine with a batch
of one; numpy views are produced only when a caller asks for them.

Differences from the reference, by construction of the B200 path:
* ``LayerStates.attn`` is None - the (L, H, n, n) attention matrix is never
  materialised (flash-style attention).
* After a DHD prefill the session has computed only the rows
  S = non-reused U selected U {n-1} (exact on those rows);
  ``prefill_states.hidden`` holds NaN on the other rows.  K/V are complete.
* ``LayerStates`` fields are materialised as float64 numpy on first access
  (device snapshots until then).
* ORACLE selection mode and the comparison strategies run on
  the device through ``select_baseline``.
"""
from __future__ import annotations

from collections.abc import Mapping
from dataclasses import dataclass, field

import numpy as np
import torch

from .engine import BatchState, Engine, RowSet
from .errors import CacheError, InputError, ParameterError
from .model import HEAD_DIM, ToyModel
from .pool import CachePool, KVArena, ReuseMap
from .selection import SelectionConfig, SelectionMode, Strategy

def get_engine(model: ToyModel, pool: CachePool | None = None, need_tokens: int = 0) -> Engine:
    """One engine per (model, pool), cached on the pool (or, for a private
    growing pool when pool is None, on the model) - nothing global keeps a
    model, pool or arena alive after the caller drops them."""
    if pool is not None:
        engines = pool.__dict__.setdefault("_engines", {})
        eng = engines.get(id(model))
        if eng is None or eng.model is not model:
            eng = engines[id(model)] = Engine(model, pool)
        return eng
    eng = getattr(model, "_private_engine", None)
    pages = KVArena(model.config, 0, model.device).pages_for(need_tokens) + 2
    if eng is None or eng.arena.free_pages < pages:
        # sessions on the previous arena keep their own engine (and arena)
        total = max(pages * 2, 64, 0 if eng is None else eng.arena.num_pages * 2)
        arena = KVArena(model.config, total, model.device)
        eng = Engine(model, CachePool(model.config, arena=arena, device=model.device))
        model._private_engine = eng
    return eng


def _pool_of(reuse: ReuseMap | None) -> CachePool | None:
    if reuse is None or not reuse.sources:
        return None
    entry = next(iter(reuse.sources.values()))[0]
    return entry.pool


def _device_hits(reuse: ReuseMap | None, n: int, device):
    slot = np.full(n, -1, dtype=np.int32)
    cand = np.full(n, -1, dtype=np.int32)
    if reuse is not None:
        for pos, (entry, c) in reuse.sources.items():
            if not 0 <= pos < n:
                raise InputError(f"reuse position {pos} outside request of length {n}")
            if not 0 <= c < entry.n_tokens:
                raise CacheError(f"cached position {c} outside entry")
            entry.check_live()
            slot[pos] = entry.slot
            cand[pos] = c
    return torch.from_numpy(slot).to(device), torch.from_numpy(cand).to(device)


class LayerStates:
    """Per-layer states (model.py:132-151); attn is None.

    The fields are float64 numpy arrays of the reference's shapes - q and
    head_out (L, H, n, d_k), k and v (L, kv_heads, n, d_k), hidden
    (L+1, n, d_model) - built on first access from device snapshots taken
    when the pass ran, so a Llama-shape prefill keeps ~1 GB of bf16/fp32 on
    the GPU instead of ~15 GB of float64 on the host unless a caller reads
    them.  Rows a partial prefill did not compute read as NaN."""

    attn = None

    def __init__(self, model: ToyModel, n: int, pos: torch.Tensor, capture, x0: torch.Tensor,
                 kv: torch.Tensor):
        self._model, self._n, self._pos = model, n, pos
        self._capture, self._x0, self._kv = capture, x0, kv       # kv: [L, 2, n, G, 128] bf16
        self._cache: dict = {}

    @property
    def n_tokens(self) -> int:
        return self._n

    def _heads(self, which: int) -> np.ndarray:
        cfg, m = self._model.config, self._model
        out = np.full((cfg.num_layers, cfg.num_heads, self._n, cfg.d_k), np.nan)
        pos = self._pos.cpu().numpy()
        for item in self._capture:
            if item[1] != "hidden":
                out[item[0]][:, pos] = m.unpad_heads(item[which]).float().permute(1, 0, 2) \
                    .cpu().numpy()
        return out

    @property
    def q(self) -> np.ndarray:
        if "q" not in self._cache:
            self._cache["q"] = self._heads(1)
        return self._cache["q"]

    @property
    def head_out(self) -> np.ndarray:
        if "head_out" not in self._cache:
            self._cache["head_out"] = self._heads(2)
        return self._cache["head_out"]

    @property
    def hidden(self) -> np.ndarray:
        if "hidden" not in self._cache:
            cfg = self._model.config
            hid = np.full((cfg.num_layers + 1, self._n, cfg.d_model), np.nan)
            pos = self._pos.cpu().numpy()
            hid[0][pos] = self._x0.double().cpu().numpy()
            for item in self._capture:
                if item[1] == "hidden":
                    hid[item[0] + 1][pos] = item[2].double().cpu().numpy()
            self._cache["hidden"] = hid
        return self._cache["hidden"]

    def _kv_host(self, which: int) -> np.ndarray:
        x = self._model.unpad_heads(self._kv[:, which])                # L, n, G, d_k
        return x.float().permute(0, 2, 1, 3).double().cpu().numpy()

    @property
    def k(self) -> np.ndarray:
        if "k" not in self._cache:
            self._cache["k"] = self._kv_host(0)
        return self._cache["k"]

    @property
    def v(self) -> np.ndarray:
        if "v" not in self._cache:
            self._cache["v"] = self._kv_host(1)
        return self._cache["v"]


def _kv_device(eng: Engine, st: BatchState, r: int, n: int) -> torch.Tensor:
    """Snapshot of request r's K/V rows [0, n): [L, 2, n, G, 128] bf16."""
    return torch.stack([torch.stack([eng.arena.rows(st.pages[r], n, layer, kv) for kv in (0, 1)])
                        for layer in range(eng.cfg.num_layers)])


def _kv_numpy(eng: Engine, st: BatchState, r: int, n: int, kv: int) -> np.ndarray:
    out = []
    for layer in range(eng.cfg.num_layers):
        rows = eng.arena.rows(st.pages[r], n, layer, kv)
        out.append(eng.model.unpad_heads(rows).float().permute(1, 0, 2).cpu().numpy())
    return np.stack(out).astype(np.float64)


def _states_from_capture(eng: Engine, st: BatchState, rows: RowSet, capture, x0) -> LayerStates:
    n = int(st.lengths[0])
    return LayerStates(eng.model, n, rows.row_pos, capture, x0, _kv_device(eng, st, 0, n))


def _normalize_recompute(recompute, L: int) -> list[set]:
    if recompute is None:
        return [set() for _ in range(L)]
    if isinstance(recompute, Mapping):
        return [set(recompute.get(layer, ())) for layer in range(L)]
    if isinstance(recompute, (list, tuple)) and recompute and \
            all(isinstance(s, (set, frozenset)) for s in recompute):
        return [set(s) for s in recompute]
    fixed = set(recompute)
    return [set(fixed) for _ in range(L)]


def _forward_session(model: ToyModel, tokens, reuse, sets, decode_capacity=64):
    """model.py:163-208 over all rows on the device (+ a live BatchState)."""
    tokens = np.asarray(tokens, dtype=np.int64)
    model.check_tokens(tokens)
    pool = _pool_of(reuse)
    eng = get_engine(model, pool, tokens.size + decode_capacity)
    st = eng.new_batch([tokens], decode_capacity)
    n = tokens.size
    st.src_slot, st.src_cand = _device_hits(reuse, n, eng.device)
    st.n_hit = np.array([int((st.src_slot >= 0).sum().item())])
    if st.n_hit[0] and pool is not None:
        eng.gather(st)
    rows = eng._rows_all(st)
    reused = st.src_slot >= 0
    per_layer = []
    for s in sets:
        rec = torch.zeros(n, dtype=torch.bool, device=eng.device)
        if s:
            rec[torch.tensor(sorted(p for p in s if 0 <= p < n), dtype=torch.long,
                             device=eng.device)] = True
        per_layer.append((~reused | rec).to(torch.uint8))
    capture = []
    x = eng._embed(st.tokens, rows)
    x0 = x.clone()
    x = eng.forward_rows(x, rows, range(eng.cfg.num_layers), eng.arena.c, st.batch_c,
                         write_kv_per_layer=per_layer, capture=capture)
    st.rows = rows
    st.hidden_last = x[-1:]
    states = _states_from_capture(eng, st, rows, capture, x0)
    return eng, st, states


def model_forward(tokens, model: ToyModel) -> LayerStates:
    eng, st, states = _forward_session(model, tokens, None, _normalize_recompute(
        None, model.config.num_layers), decode_capacity=0)
    eng.release(st)
    return states


def model_forward_with_reuse(tokens, model: ToyModel, reuse: ReuseMap | None,
                             recompute=None) -> LayerStates:
    eng, st, states = _forward_session(model, tokens, reuse, _normalize_recompute(
        recompute, model.config.num_layers), decode_capacity=0)
    eng.release(st)
    return states


@dataclass
class StepStates:
    """Per-step output (engine.py:38-44); q/attn are not materialised."""

    q: None
    attn: None
    hidden_out: np.ndarray


class ReuseSession:
    """Mutable device K/V cache of one request (engine.py:47-171)."""

    def __init__(self, model: ToyModel, tokens, reuse=None, recompute=None,
                 _engine_state=None, decode_capacity: int = 256):
        cfg = model.config
        self.model = model
        self.tokens = [int(t) for t in np.asarray(tokens, dtype=np.int64)]
        self.n_prefill = len(self.tokens)
        sets = _normalize_recompute(recompute, cfg.num_layers)
        if _engine_state is None:
            eng, st, states = _forward_session(model, tokens, reuse, sets, decode_capacity)
            self.prefill_states = states
        else:
            eng, st, self.prefill_states = _engine_state
        self.engine, self.state = eng, st
        self.reused = set() if reuse is None else set(reuse.sources)
        self.recomputed = [set(s) & self.reused for s in sets]
        self.probe_layer = 1 if cfg.num_layers >= 2 else 0
        elig = np.zeros(self.n_prefill, dtype=np.uint8)
        common = set.intersection(*self.recomputed) if self.recomputed else set()
        for p in self.reused - common:
            elig[p] = 1
        st.eligible = torch.from_numpy(elig).to(eng.device)
        st.tokens_host = [list(self.tokens)]

    @property
    def n_tokens(self) -> int:
        return len(self.tokens)

    @property
    def k(self) -> np.ndarray:
        return _kv_numpy(self.engine, self.state, 0, self.n_tokens, 0)

    @property
    def v(self) -> np.ndarray:
        return _kv_numpy(self.engine, self.state, 0, self.n_tokens, 1)

    def _grow(self, extra: int = 1):
        st, eng = self.state, self.engine
        need = self.n_tokens + extra
        if need <= st.capacity[0]:
            return
        add = eng.arena.pages_for(need + 256) - len(st.pages[0])
        st.pages[0] = st.pages[0] + eng.arena.alloc(add)
        bt = np.array([st.pages[0]], dtype=np.int32)
        st.block_table = torch.from_numpy(bt).to(eng.device)
        st.batch_c.block_table = st.block_table.data_ptr()
        st.batch_c.max_pages = bt.shape[1]
        st.capacity = np.array([len(st.pages[0]) * eng.arena.page_size])
        st._keep = (st.req_off, st.block_table)

    def append(self, token_id: int) -> StepStates:
        """engine.py:114-121: run the token through all layers, grow the cache."""
        self.model.check_tokens(np.array([token_id], dtype=np.int64))
        self._grow(1)
        h, _ = self.engine.decode_step(self.state, [int(token_id)], 0)
        self.tokens.append(int(token_id))
        return StepStates(None, None, h[0].double().cpu().numpy())

    def recompute_positions(self, positions) -> None:
        """engine.py:123-138 as one layer-batched pass."""
        pos = sorted(set(int(p) for p in positions))
        for p in pos:
            if not 0 <= p < self.n_tokens:
                raise InputError(f"position {p} outside sequence of {self.n_tokens}")
        if not pos:
            return
        eng, st = self.engine, self.state
        rows = RowSet(len(pos), torch.arange(len(pos), dtype=torch.int32, device=eng.device),
                      torch.zeros(len(pos), dtype=torch.int32, device=eng.device),
                      torch.tensor(pos, dtype=torch.int32, device=eng.device), None,
                      np.array([0, len(pos)], dtype=np.int64))
        tok = torch.tensor([self.tokens[p] for p in pos], dtype=torch.int64, device=eng.device)
        x = eng._embed(tok, rows)
        x = eng.forward_rows(x, rows, range(eng.cfg.num_layers), eng.arena.c, st.batch_c,
                             decode=True, max_kv=int(st.capacity.max()))
        elig = st.eligible
        for p in pos:
            if p in self.reused:
                for s in self.recomputed:
                    s.add(p)
            if p < elig.numel():
                elig[p] = 0

    def delta_v_probe(self) -> np.ndarray:
        """engine.py:140-148: cache V at the probe layer minus its exact value."""
        eng, st = self.engine, self.state
        _, _, v_true = eng._probe(st, write_k=False)
        cache_v = eng.arena.rows(st.pages[0], self.n_tokens, self.probe_layer, 1)
        delta = torch.zeros_like(cache_v, dtype=torch.float32)
        n = self.n_prefill
        delta[:n] = cache_v[:n].float() - v_true.float()
        return eng.model.unpad_heads(delta).permute(1, 0, 2).double().cpu().numpy()

    def query_rows_probe(self, token_id: int) -> np.ndarray:
        """engine.py:150-171 (the new token's own layer-0 row is written at
        position n_tokens, beyond the context; append overwrites it with the
        same value)."""
        self._grow(1)
        q = self.engine.probe_query(self.state, np.array([int(token_id)]))
        return self.model.unpad_heads(q[0]).double().cpu().numpy()


@dataclass
class PrefillResult:
    session: ReuseSession
    recompute_sets: list
    selected: tuple = ()
    eligible: set = field(default_factory=set)


def prefill_with_selection(model: ToyModel, tokens, reuse, config: SelectionConfig,
                           ref_states=None, decode_capacity: int = 256) -> PrefillResult:
    """engine.py:217-243 (PRACTICAL): probe, DHD select, partial prefill."""
    reused = sorted(reuse.sources) if reuse is not None else []
    if not reused:
        session = ReuseSession(model, tokens, reuse, decode_capacity=decode_capacity)
        return PrefillResult(session, session.recomputed)
    if config.mode is SelectionMode.ORACLE:
        return _oracle_prefill(model, tokens, reuse, config, ref_states, decode_capacity)
    if Strategy(config.strategy) is not Strategy.ATTENTION_WEIGHTED:
        return _practical_baseline(model, tokens, reuse, config, decode_capacity)
    tokens = np.asarray(tokens, dtype=np.int64)
    model.check_tokens(tokens)
    pool = _pool_of(reuse)
    eng = get_engine(model, pool)
    st = eng.new_batch([tokens], decode_capacity)
    st.src_slot, st.src_cand = _device_hits(reuse, tokens.size, eng.device)
    st.n_hit = np.array([len(reused)])
    eng.gather(st)
    eng.probe_and_select(st, config.ratio)
    rows = eng.build_rows(st, st.selected)
    capture = []
    x = eng._embed(st.tokens, rows)
    x0 = x.clone()
    x = eng.forward_rows(x, rows, range(eng.cfg.num_layers), eng.arena.c, st.batch_c,
                         capture=capture)
    st.rows = rows
    st.hidden_last = x[-1:]
    states = _states_from_capture(eng, st, rows, capture, x0)
    selected = tuple(int(i) for i in torch.nonzero(st.selected).flatten().cpu().tolist())
    session = ReuseSession(model, tokens, reuse, set(selected), _engine_state=(eng, st, states))
    eligible = set(reused) - set(selected)
    return PrefillResult(session, session.recomputed, selected, eligible)


def _probe_states(eng: Engine, st: BatchState):
    """The perturbed probe (engine.py:195-207) as host arrays:
    (q, k_true, v_true, k_pert, v_pert), heads unpadded, kv at kv_heads."""
    cfg, m = eng.cfg, eng.model
    n = int(st.lengths[0])
    k_true = torch.empty(n, cfg.kv_heads, 128, dtype=torch.bfloat16, device=eng.device)
    _, q1, v_true = eng._probe(st, k_out=k_true)
    p = eng.probe_layer

    def host(x):                                             # [n, heads, 128] -> (heads, n, d)
        return m.unpad_heads(x).float().permute(1, 0, 2).double().cpu().numpy()

    kp = host(eng.arena.rows(st.pages[0], n, p, 0))
    vp = host(eng.arena.rows(st.pages[0], n, p, 1))
    return host(q1), host(k_true), host(v_true), kp, vp


def _restrict(delta: np.ndarray, keep) -> np.ndarray:
    """engine.py:210-214: zero every row outside `keep`."""
    out = np.zeros_like(delta)
    idx = sorted(keep)
    out[:, idx, :] = delta[:, idx, :]
    return out


def _practical_baseline(model, tokens, reuse, config, decode_capacity):
    """engine.py:233-243 PRACTICAL mode with a comparison strategy: the
    layer-1 probe's deviations scored by select_baseline (F4), the same set
    recomputed at every layer."""
    from .selection import select_baseline
    tokens = np.asarray(tokens, dtype=np.int64)
    model.check_tokens(tokens)
    reused = sorted(reuse.sources)
    pool = _pool_of(reuse)
    eng = get_engine(model, pool)
    st = eng.new_batch([tokens], 0)
    st.src_slot, st.src_cand = _device_hits(reuse, tokens.size, eng.device)
    eng.gather(st)
    qp, kt, vt, kp, vp = _probe_states(eng, st)
    eng.release(st)
    keep = set(reused)
    result = select_baseline(config.strategy, qp, kt, vt, _restrict(kp - kt, keep),
                             _restrict(vp - vt, keep), reused, config)
    selected = result.indices
    session = ReuseSession(model, tokens, reuse, set(selected), decode_capacity=decode_capacity)
    return PrefillResult(session, session.recomputed, selected, set(reused) - set(selected))


def _oracle_prefill(model, tokens, reuse, config, ref_states, decode_capacity):
    """engine.py:245-285 ORACLE mode: per layer, the true deviation of the
    perturbed K/V against a fresh reference pass (ref_states) is scored by
    the configured strategy (select_baseline) and that layer's selected rows
    are restored to fresh before the layer's attention runs."""
    from .selection import select_baseline
    if ref_states is None:
        raise ParameterError("oracle-mode prefill needs reference layer states")
    tokens = np.asarray(tokens, dtype=np.int64)
    model.check_tokens(tokens)
    reused = sorted(reuse.sources)
    keep = set(reused)
    cfg, m = model.config, model
    pool = _pool_of(reuse)
    n = tokens.size
    eng = get_engine(model, pool, n + decode_capacity)
    st = eng.new_batch([tokens], decode_capacity)
    st.src_slot, st.src_cand = _device_hits(reuse, n, eng.device)
    st.n_hit = np.array([len(reused)])
    eng.gather(st)                                    # cached (re-aligned) K/V, every layer
    rows = eng._rows_all(st)
    dev, H, G = eng.device, cfg.num_heads, cfg.kv_heads
    fresh_rows = (st.src_slot < 0).to(torch.uint8)
    q = torch.empty(n, H, 128, dtype=torch.bfloat16, device=dev)
    o = torch.empty_like(q)
    x = eng._embed(st.tokens, rows)
    x0 = x.clone()
    capture, sets = [], []

    def host(t):
        return m.unpad_heads(t).float().permute(1, 0, 2).double().cpu().numpy()

    for layer in range(cfg.num_layers):
        qkv = eng._qkv(x, layer)
        eng._scatter(qkv, rows, layer, eng.arena.c, st.batch_c, q, write_kv=fresh_rows)
        kp = host(eng.arena.rows(st.pages[0], n, layer, 0))
        vp = host(eng.arena.rows(st.pages[0], n, layer, 1))
        dk = _restrict(kp - ref_states.k[layer], keep)
        dv = _restrict(vp - ref_states.v[layer], keep)
        result = select_baseline(config.strategy, host(q), ref_states.k[layer],
                                 ref_states.v[layer], dk, dv, reused, config)
        sel = set(result.indices)
        if sel:
            mask = torch.zeros(n, dtype=torch.uint8, device=dev)
            mask[torch.as_tensor(sorted(sel), dtype=torch.long, device=dev)] = 1
            eng._scatter(qkv, rows, layer, eng.arena.c, st.batch_c, q, write_kv=mask)
        sets.append(sel)
        eng._attention(q, rows, layer, eng.arena.c, st.batch_c, o)
        capture.append((layer, q.clone(), o.clone()))
        eng._out_proj(x, o, layer)
        capture.append((layer, "hidden", x.clone()))
    st.rows = rows
    st.hidden_last = x[-1:]
    states = _states_from_capture(eng, st, rows, capture, x0)
    session = ReuseSession(model, tokens, reuse, sets, _engine_state=(eng, st, states))
    eligible = keep - set.intersection(*sets) if sets else set()
    return PrefillResult(session, session.recomputed, tuple(sorted(set.union(*sets))), eligible)


@dataclass
class GenerationResult:
    """engine.py:288-295; ``chosen`` (positions recomputed per step) is an
    addition the reference records only through recompute_positions."""

    step_deviation: list
    recompute_counts: list
    chosen: list = field(default_factory=list)

    @property
    def cumulative_deviation(self) -> float:
        return float(sum(self.step_deviation))


def run_generation(session: ReuseSession, ref_session: ReuseSession, decode_tokens,
                   n_extra: int) -> GenerationResult:
    """engine.py:298-328: per token, D3 selection + recompute + append on the
    session, append on the reference session, ||h - h_ref||."""
    deviations, counts, chosen_steps = [], [], []
    for tok in decode_tokens:
        tok = int(tok)
        session._grow(1)
        h, chosen = session.engine.decode_step(session.state, [tok], n_extra)
        for p in chosen[0]:
            if p in session.reused:
                for s in session.recomputed:
                    s.add(p)
        session.tokens.append(tok)
        ref = ref_session.append(tok)
        deviations.append(float(np.linalg.norm(h[0].double().cpu().numpy() - ref.hidden_out)))
        counts.append(len(chosen[0]))
        chosen_steps.append(list(chosen[0]))
    return GenerationResult(deviations, counts, chosen_steps)
