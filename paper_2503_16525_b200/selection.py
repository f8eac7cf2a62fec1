"""Recompute-token selection for both serving phases, on the GPU.

Drop-in for reference pkg/src/kvlab/selection.py: ``Strategy``,
``SelectionMode``, ``SelectionConfig`` (:37-52, budget with the exact
IEEE-double ceil), ``SelectionResult``, ``select_prefill`` (:69-77, D1 + D2
radix top-B) and ``select_decode_step`` (:80-105, D3).  ``select_baseline``
(:133-186) runs all five strategies: the hot path's ATTENTION_WEIGHTED and
the comparison baselines of the SURVEY's row F4 (MAGNITUDE / POSITIONAL /
RANDOM / IDEAL) with device scoring and the kvs_topk_select top-B.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from enum import Enum

import numpy as np
import torch

from . import _native as N
from ._scratch import Scratch, as_heads, dense_rows
from .deviation import alpha_scores
from .errors import ParameterError, ShapeError


class Strategy(str, Enum):
    ATTENTION_WEIGHTED = "attention_weighted"
    MAGNITUDE = "magnitude"
    POSITIONAL = "positional"
    RANDOM = "random"
    IDEAL = "ideal"


class SelectionMode(str, Enum):
    ORACLE = "oracle"
    PRACTICAL = "practical"


@dataclass(frozen=True)
class SelectionConfig:
    ratio: float = 0.2
    n_extra: int = 3
    mode: SelectionMode = SelectionMode.PRACTICAL
    strategy: Strategy = Strategy.ATTENTION_WEIGHTED
    seed: int = 0

    def __post_init__(self):
        if not 0.0 < self.ratio <= 1.0:
            raise ParameterError(f"ratio must lie in (0, 1], got {self.ratio}")
        if self.n_extra < 0:
            raise ParameterError(f"n_extra must be >= 0, got {self.n_extra}")

    def budget(self, n_reused: int) -> int:
        return min(math.ceil(self.ratio * n_reused), n_reused)


@dataclass
class SelectionResult:
    """Chosen token positions (ascending) and the scores that ranked them."""

    indices: tuple[int, ...]
    scores: np.ndarray


def select_prefill(q, k, delta_v, reused, config: SelectionConfig,
                   causal: bool = True) -> SelectionResult:
    """Rank reused tokens by attention-weighted value deviation, keep top r."""
    reused = sorted(set(int(i) for i in reused))
    if not reused:
        raise ParameterError("reused set is empty")
    n = as_heads(k).shape[1]
    if reused[0] < 0 or reused[-1] >= n:
        raise ParameterError("reused position outside the sequence")
    mask = np.zeros(n, dtype=bool)
    mask[reused] = True
    scores, _, _, sel = alpha_scores(q, k, delta_v, causal, mask, config.budget(len(reused)))
    return SelectionResult(tuple(int(i) for i in np.nonzero(sel)[0]), scores)


_dws = N.Workspace()
_sws = N.Workspace()


def _sel_ws(dev, n: int = 1):
    return _sws.get(N.ws_bytes("kvs_dhd_select_workspace", n, 1), dev, zero=True)


def select_decode_step(q_t, k, delta_v, eligible, n_extra: int) -> SelectionResult:
    """selection.py:80-105 via D3 (kvs_dhd_decode_select)."""
    q_t = np.atleast_2d(np.asarray(q_t, float))
    k = np.asarray(k, float)
    delta_v = np.asarray(delta_v, float)
    if k.ndim == 2:
        k = k[None]
        delta_v = delta_v[None]
    if q_t.shape[-1] != k.shape[-1] or q_t.shape[0] % k.shape[0] != 0:
        raise ShapeError(f"q_t {q_t.shape} incompatible with k {k.shape}")
    if delta_v.shape != k.shape:
        raise ShapeError(f"delta_v {delta_v.shape} does not match k {k.shape}")
    n = k.shape[1]
    eligible = sorted(set(int(i) for i in eligible))
    if not eligible or n_extra <= 0:
        return SelectionResult((), np.zeros(n))
    k, delta_v = as_heads(k), as_heads(delta_v)
    N.load()
    dev = torch.device("cuda", torch.cuda.current_device())
    H, d = q_t.shape[0], q_t.shape[1]
    sc = Scratch(k, delta_v, dev)
    zeros_v = torch.zeros(n, k.shape[0], 128, dtype=torch.bfloat16, device=dev)
    alpha0 = torch.zeros(n, dtype=torch.float32, device=dev)
    slot = torch.zeros(n, dtype=torch.int32, device=dev)
    bud = torch.zeros(1, dtype=torch.int32, device=dev)
    dv = torch.empty(n, dtype=torch.float32, device=dev)
    tmp = torch.empty(n, dtype=torch.float32, device=dev)
    tsel = torch.empty(n, dtype=torch.uint8, device=dev)
    N.call("kvs_dhd_select", zeros_v.data_ptr(), alpha0.data_ptr(), slot.data_ptr(), 0, sc.arena,
           sc.batch, bud.data_ptr(), dv.data_ptr(), tmp.data_ptr(), tsel.data_ptr(), _sel_ws(dev, n).data_ptr(),
           _sel_ws(dev, n).numel(), N.stream_ptr())
    qd = dense_rows(q_t[:, None, :], dev)                 # [1, H, 128]
    elig = np.zeros(n, dtype=np.uint8)
    elig[[e for e in eligible if 0 <= e < n]] = 1
    elig_t = torch.from_numpy(elig).to(dev)
    ctx = torch.tensor([n], dtype=torch.int32, device=dev)
    chosen = torch.empty(1, n_extra, dtype=torch.int32, device=dev)
    nch = torch.zeros(1, dtype=torch.int32, device=dev)
    scores = torch.zeros(1, n, dtype=torch.float32, device=dev)
    ws = _dws.get(N.ws_bytes("kvs_dhd_decode_select_workspace", 1, H, n), dev, zero=True)
    N.call("kvs_dhd_decode_select", qd.data_ptr(), H, ctx.data_ptr(), n, dv.data_ptr(),
           elig_t.data_ptr(), 0, sc.arena, sc.batch, n_extra, 1.0 / math.sqrt(d),
           chosen.data_ptr(), nch.data_ptr(), scores.data_ptr(), ws.data_ptr(), ws.numel(),
           N.stream_ptr())
    c = int(nch.item())
    return SelectionResult(tuple(int(x) for x in chosen[0, :c].cpu().tolist()),
                           scores[0].double().cpu().numpy())


def _spans(positions: list[int]) -> list[list[int]]:
    """Contiguous runs of an ascending position list (selection.py:108-116)."""
    runs: list[list[int]] = []
    for p in positions:
        if runs and p == runs[-1][-1] + 1:
            runs[-1].append(p)
        else:
            runs.append([p])
    return runs


def _positional_selection(reused: list[int], config: SelectionConfig) -> tuple[int, ...]:
    """Leading positions of each reused span, trimmed/padded to the budget
    (selection.py:119-130); pure index logic on the host."""
    budget = config.budget(len(reused))
    chosen: list[int] = []
    for span in _spans(reused):
        chosen.extend(span[: math.ceil(config.ratio * len(span))])
    if len(chosen) > budget:
        chosen = sorted(chosen)[:budget]
    elif len(chosen) < budget:
        taken = set(chosen)
        rest = [p for p in reused if p not in taken]
        chosen.extend(rest[: budget - len(chosen)])
    return tuple(sorted(chosen))


def _device_top(scores: torch.Tensor, reused: list[int], budget: int) -> tuple[int, ...]:
    """_take_top (selection.py:63-66) on the device: kvs_topk_select over the
    reused positions, score descending, position ascending."""
    dev, n = scores.device, scores.numel()
    cand = torch.full((n,), -1, dtype=torch.int32, device=dev)
    cand[torch.as_tensor(reused, dtype=torch.long, device=dev)] = 0
    off = torch.tensor([0, n], dtype=torch.int64, device=dev)
    bud = torch.tensor([budget], dtype=torch.int32, device=dev)
    sel = torch.zeros(n, dtype=torch.uint8, device=dev)
    N.call("kvs_topk_select", scores.data_ptr(), cand.data_ptr(), off.data_ptr(), 1, n,
           bud.data_ptr(), sel.data_ptr(), N.stream_ptr())
    return tuple(int(i) for i in torch.nonzero(sel).flatten().cpu().tolist())


def select_baseline(strategy, q, k, v, delta_k, delta_v, reused, config: SelectionConfig,
                    causal: bool = True) -> SelectionResult:
    """selection.py:133-186: run one of the comparison strategies over the
    same reuse scenario.  ``k``/``v`` are the fresh matrices and
    ``delta_k``/``delta_v`` the cached-minus-fresh increments (rows outside
    ``reused`` zero), (H, n, d) or (n, d).

    ATTENTION_WEIGHTED: D1 + D2 against the perturbed keys (as served).
    MAGNITUDE: sum |dv| + |dk| on the device, kvs_topk_select.
    POSITIONAL: span heads (host index logic).
    RANDOM: the reference's Philox(key=seed) uniforms, kvs_topk_select.
    IDEAL: kvs_ideal_scores (leave-one-in deviation in closed form),
    kvs_topk_select."""
    try:
        strategy = Strategy(strategy)
    except ValueError:
        raise ParameterError(f"unknown strategy: {strategy!r}") from None
    reused = sorted(set(int(i) for i in reused))
    if not reused:
        raise ParameterError("reused set is empty")
    if strategy is Strategy.ATTENTION_WEIGHTED:
        kp = np.asarray(k, float) + np.asarray(delta_k, float)
        return select_prefill(q, kp, delta_v, reused, config, causal=causal)
    qh, kh, vh = as_heads(q), as_heads(k), as_heads(v)
    dkh, dvh = as_heads(delta_k), as_heads(delta_v)
    n = kh.shape[1]
    budget = config.budget(len(reused))
    if strategy is Strategy.POSITIONAL:
        return SelectionResult(_positional_selection(reused, config), np.zeros(n))
    dev = torch.device("cuda", torch.cuda.current_device())
    N.load()
    if strategy is Strategy.MAGNITUDE:
        dk_t = torch.as_tensor(dkh, dtype=torch.float32, device=dev)
        dv_t = torch.as_tensor(dvh, dtype=torch.float32, device=dev)
        scores = (dv_t.abs().sum(dim=(0, 2)) + dk_t.abs().sum(dim=(0, 2))).contiguous()
    elif strategy is Strategy.RANDOM:
        gen = np.random.Generator(np.random.Philox(key=config.seed))
        host = np.zeros(n)
        host[reused] = gen.uniform(size=len(reused))
        scores = torch.as_tensor(host, dtype=torch.float32, device=dev)
    else:                                                       # IDEAL
        H, G, d = qh.shape[0], kh.shape[0], qh.shape[2]
        t = [torch.as_tensor(np.ascontiguousarray(x), dtype=torch.float32, device=dev)
             for x in (qh, kh, vh, dkh, dvh)]
        scores = torch.empty(n, dtype=torch.float32, device=dev)
        ws = torch.empty(N.ws_bytes("kvs_ideal_scores_workspace", H, n, d), dtype=torch.uint8,
                         device=dev)
        N.call("kvs_ideal_scores", *(x.data_ptr() for x in t), H, G, n, d, 1 if causal else 0,
               1.0 / math.sqrt(d), scores.data_ptr(), ws.data_ptr(), ws.numel(), N.stream_ptr())
        mask = torch.zeros(n, dtype=torch.bool, device=dev)
        mask[torch.as_tensor(reused, dtype=torch.long, device=dev)] = True
        scores = torch.where(mask, scores, torch.zeros_like(scores))
    indices = _device_top(scores, reused, budget)
    return SelectionResult(indices, scores.double().cpu().numpy())
