"""Recompute-token selection for both serving phases, on the GPU.

Drop-in for reference pkg/src/kvlab/selection.py: ``Strategy``,
``SelectionMode``, ``SelectionConfig`` (:37-52, budget with the exact
IEEE-double ceil), ``SelectionResult``, ``select_prefill`` (:69-77, D1 + D2
radix top-B) and ``select_decode_step`` (:80-105, D3).  ``select_baseline``
keeps the ATTENTION_WEIGHTED branch the hot path uses (:156-157); the
comparison baselines (MAGNITUDE/POSITIONAL/RANDOM/IDEAL) are the SURVEY's
next row F4 and raise ParameterError here.
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


def _sel_ws(dev):
    return _sws.get(N.ws_bytes("kvs_dhd_select_workspace", 1, 1), dev, zero=True)


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
           sc.batch, bud.data_ptr(), dv.data_ptr(), tmp.data_ptr(), tsel.data_ptr(), _sel_ws(dev).data_ptr(),
           _sel_ws(dev).numel(), N.stream_ptr())
    qd = dense_rows(q_t[:, None, :], dev)                 # [1, H, 128]
    elig = np.zeros(n, dtype=np.uint8)
    elig[[e for e in eligible if 0 <= e < n]] = 1
    elig_t = torch.from_numpy(elig).to(dev)
    ctx = torch.tensor([n], dtype=torch.int32, device=dev)
    chosen = torch.empty(1, n_extra, dtype=torch.int32, device=dev)
    nch = torch.zeros(1, dtype=torch.int32, device=dev)
    scores = torch.zeros(1, n, dtype=torch.float32, device=dev)
    ws = _dws.get(N.ws_bytes("kvs_dhd_decode_select_workspace", 1, H, n), dev)
    N.call("kvs_dhd_decode_select", qd.data_ptr(), H, ctx.data_ptr(), n, dv.data_ptr(),
           elig_t.data_ptr(), 0, sc.arena, sc.batch, n_extra, 1.0 / math.sqrt(d),
           chosen.data_ptr(), nch.data_ptr(), scores.data_ptr(), ws.data_ptr(), ws.numel(),
           N.stream_ptr())
    c = int(nch.item())
    return SelectionResult(tuple(int(x) for x in chosen[0, :c].cpu().tolist()),
                           scores[0].double().cpu().numpy())


def select_baseline(strategy, q, k, v, delta_k, delta_v, reused, config: SelectionConfig,
                    causal: bool = True) -> SelectionResult:
    """selection.py:133-186, ATTENTION_WEIGHTED branch (scores against the
    perturbed keys k + delta_k, as served)."""
    try:
        strategy = Strategy(strategy)
    except ValueError:
        raise ParameterError(f"unknown strategy: {strategy!r}") from None
    if strategy is not Strategy.ATTENTION_WEIGHTED:
        raise ParameterError(f"strategy {strategy.value} is a comparison baseline, not on the "
                             "device hot path (SURVEY.md F4)")
    k = np.asarray(k, float) + np.asarray(delta_k, float)
    return select_prefill(q, k, delta_v, reused, config, causal=causal)
