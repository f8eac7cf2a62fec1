"""Drop-in replacement for the reference's compiled matcher ``kvlab._matchcore``.

Same two functions and signatures as pkg/src/kvlab/_matchcore.pyx:16 and :37
(int64 token buffers, window size, base, modulus), backed by the CUDA kernels
R1/R2 through the C ABI (kvs_window_hashes, kvs_match_pairs).  Placed as
``kvlab/_matchcore`` the reference's own matcher tests
select and exercise it unchanged.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _native as N
from .matching import HashParams, match_pairs_device, window_hashes_device


class _Params:
    """HashParams without the primality re-check (the caller validated)."""

    def __init__(self, w, b, m):
        self.window_size, self.base, self.modulus = int(w), int(b), int(m)


def _dev():
    N.load()
    return torch.device("cuda", torch.cuda.current_device())


def window_hashes(tokens, w: int, b: int, m: int):
    arr = np.ascontiguousarray(np.asarray(tokens, dtype=np.int64))
    if arr.shape[0] < w:
        return np.empty(0, dtype=np.uint64)
    t = torch.from_numpy(arr).to(_dev())
    return window_hashes_device(t, _Params(w, b, m)).cpu().numpy().astype(np.uint64)


def match_pairs(target, candidate, w: int, b: int, m: int):
    t = np.ascontiguousarray(np.asarray(target, dtype=np.int64))
    c = np.ascontiguousarray(np.asarray(candidate, dtype=np.int64))
    if t.shape[0] < w or c.shape[0] < w:
        return [], []
    dev = _dev()
    tm, cm, cnt = match_pairs_device(torch.from_numpy(t).to(dev), torch.from_numpy(c).to(dev),
                                     _Params(w, b, m))
    k = int(cnt.item())
    return tm[:k].cpu().tolist(), cm[:k].cpu().tolist()


__all__ = ["window_hashes", "match_pairs", "HashParams"]
