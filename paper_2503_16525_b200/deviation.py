"""Attention-output deviation scores on the GPU.

Drop-in for ``v_impact_scores`` (reference pkg/src/kvlab/deviation.py:96-115):
score_i = colsum(causal softmax(q k^T / sqrt(d)))_i averaged over query heads
times ||delta_v_i||_1 summed over heads.  D1 (kvs_dhd_alpha, tcgen05) computes
the attention mass, D2's dv-L1 pass (kvs_dhd_select) the value deviation.
GQA extension: q may have a multiple of k's head count.

The paper-analysis functions of the reference module (delta_h_first_order,
k_impact_scores, impact_overlap, layer_retention) are outside the hot path
 and are not provided.
"""
from __future__ import annotations

import math

import numpy as np
import torch

from . import _native as N
from ._scratch import Scratch, as_heads, dense_rows
from .errors import ParameterError, ShapeError

_ws = N.Workspace()
_sws = N.Workspace()


def _sel_ws(dev, n: int = 1):
    return _sws.get(N.ws_bytes("kvs_dhd_select_workspace", n, 1), dev, zero=True)


def _dev():
    N.load()
    return torch.device("cuda", torch.cuda.current_device())


def _check(q, k, dv):
    if q.shape[1:] != k.shape[1:] or q.shape[0] % k.shape[0] != 0:
        raise ShapeError(f"q {q.shape} and k {k.shape} differ")
    if dv.shape != k.shape:
        raise ShapeError(f"delta_v {dv.shape} does not match k {k.shape}")


def alpha_scores(q, k, delta_v, causal: bool = True, reused_mask=None, budget: int = 0):
    """Run D1 + D2 on arrays; returns (scores, dv_l1, alpha, selected) as numpy."""
    q, k, dv = as_heads(q), as_heads(k), as_heads(delta_v)
    _check(q, k, dv)
    dev = _dev()
    H, n, d = q.shape
    sc = Scratch(k, dv, dev)
    qd = dense_rows(q, dev)
    alpha = torch.empty(n, dtype=torch.float32, device=dev)
    ws = _ws.get(N.ws_bytes("kvs_dhd_alpha_workspace", n, H, k.shape[0]), dev)
    N.call("kvs_dhd_alpha", qd.data_ptr(), H, 1 if causal else 0, 0, sc.arena, sc.batch,
           sc.row_pos.data_ptr(), sc.tiles[0].data_ptr(), sc.tiles[1].data_ptr(),
           sc.tiles[2].data_ptr(), sc.n_tiles, sc.kv_len.data_ptr(), 1.0 / math.sqrt(d),
           alpha.data_ptr(), ws.data_ptr(), ws.numel(), N.stream_ptr())
    zeros_v = torch.zeros(n, k.shape[0], 128, dtype=torch.bfloat16, device=dev)
    dv_l1 = torch.empty(n, dtype=torch.float32, device=dev)
    score = torch.empty(n, dtype=torch.float32, device=dev)
    sel = torch.zeros(n, dtype=torch.uint8, device=dev)

    sws = _sws.get(N.ws_bytes("kvs_dhd_select_workspace", n, 1), dev, zero=True)

    def select(slot, b):
        bud = torch.tensor([b], dtype=torch.int32, device=dev)
        N.call("kvs_dhd_select", zeros_v.data_ptr(), alpha.data_ptr(), slot.data_ptr(), 0,
               sc.arena, sc.batch, bud.data_ptr(), dv_l1.data_ptr(), score.data_ptr(),
               sel.data_ptr(), sws.data_ptr(), sws.numel(), N.stream_ptr())

    if reused_mask is not None:
        # selection restricted to the reused rows (selection.py:63-66) ...
        select(torch.from_numpy(np.where(reused_mask, 0, -1).astype(np.int32)).to(dev), budget)
        picked = sel.clone()
    # ... while the returned scores cover every row (deviation.py:96-115)
    select(torch.zeros(n, dtype=torch.int32, device=dev), 0)
    if reused_mask is not None:
        sel = picked
    return (score.double().cpu().numpy(), dv_l1.double().cpu().numpy(),
            alpha.double().cpu().numpy(), sel.cpu().numpy().astype(bool))


def v_impact_scores(q, k, delta_v, causal: bool = True) -> np.ndarray:
    """deviation.py:96-115 on the GPU (bf16 operands, fp32 accumulation)."""
    scores, _, _, _ = alpha_scores(q, k, delta_v, causal)
    return scores


def top_indices(scores, ratio: float) -> set[int]:
    """deviation.py:147-155: top ceil(ratio*n) scores, ties to the lower index."""
    scores = np.asarray(scores, float)
    n = scores.shape[0]
    if not 0.0 < ratio <= 1.0:
        raise ParameterError(f"ratio must lie in (0, 1], got {ratio}")
    count = min(math.ceil(ratio * n), n)
    order = sorted(range(n), key=lambda i: (-scores[i], i))
    return set(order[:count])
