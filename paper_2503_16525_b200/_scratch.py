"""Upload plain (heads, n, d) arrays into a one-layer scratch arena so the
array-level drop-ins (v_impact_scores, select_prefill, select_decode_step)
run on exactly the same kernels as the engine.  Head dims < 128 are
zero-padded (dot products, L1 norms and softmax are unchanged by zeros)."""
from __future__ import annotations

import numpy as np
import torch

from . import _native as N
from .errors import ShapeError
from .model import HEAD_DIM
from .pool import PAGE_SIZE


def as_heads(x) -> np.ndarray:
    x = np.asarray(x, dtype=np.float64)
    if x.ndim == 2:
        x = x[None]
    if x.ndim != 3:
        raise ShapeError(f"expected (heads, n, d) or (n, d), got shape {x.shape}")
    if x.shape[-1] > HEAD_DIM:
        raise ShapeError(f"head dim {x.shape[-1]} exceeds {HEAD_DIM}")
    return x


def dense_rows(x: np.ndarray, device) -> torch.Tensor:
    """(heads, n, d) -> bf16 [n, heads, 128] zero-padded."""
    h, n, d = x.shape
    out = torch.zeros(n, h, HEAD_DIM, dtype=torch.float32, device=device)
    out[:, :, :d] = torch.from_numpy(np.ascontiguousarray(x.transpose(1, 0, 2))).to(device)
    return out.to(torch.bfloat16).contiguous()


class Scratch:
    """One request, one layer: K (and V) rows in arena pages."""

    def __init__(self, k: np.ndarray, v: np.ndarray | None, device):
        g, n, d = k.shape
        pages = (n + PAGE_SIZE - 1) // PAGE_SIZE
        data = torch.zeros(pages, 1, 2, PAGE_SIZE, g, HEAD_DIM, dtype=torch.float32,
                           device=device)
        kk = torch.zeros(pages * PAGE_SIZE, g, HEAD_DIM, device=device)
        kk[:n, :, :d] = torch.from_numpy(np.ascontiguousarray(k.transpose(1, 0, 2))).to(device)
        data[:, 0, 0] = kk.view(pages, PAGE_SIZE, g, HEAD_DIM)
        if v is not None:
            vv = torch.zeros(pages * PAGE_SIZE, g, HEAD_DIM, device=device)
            vv[:n, :, :d] = torch.from_numpy(np.ascontiguousarray(v.transpose(1, 0, 2))).to(device)
            data[:, 0, 1] = vv.view(pages, PAGE_SIZE, g, HEAD_DIM)
        self.data = data.to(torch.bfloat16).contiguous()
        self.n, self.g = n, g
        self.req_off = torch.tensor([0, n], dtype=torch.int64, device=device)
        self.block_table = torch.arange(pages, dtype=torch.int32, device=device).view(1, pages)
        self.kv_len = torch.tensor([n], dtype=torch.int32, device=device)
        self.arena = N.KVArena(self.data.data_ptr(), pages, 1, g, HEAD_DIM, PAGE_SIZE)
        self.batch = N.Batch(1, n, self.req_off.data_ptr(), self.block_table.data_ptr(), pages)
        pos = np.arange(n, dtype=np.int32)
        self.row_pos = torch.from_numpy(pos).to(device)
        t0 = np.arange(0, n, 128, dtype=np.int32)
        self.tiles = torch.from_numpy(np.stack([np.zeros_like(t0), t0,
                                                np.minimum(128, n - t0)]).astype(np.int32)).to(device)
        self.n_tiles = len(t0)
