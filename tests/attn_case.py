"""Shared A1 attention case builder for the kernel parity test and the
micro-benchmark: a paged arena holding random K/V for R requests, random Q
for a row set S (every request's rows in ascending position order, either
all positions or a scattered subset like a DHD partial prefill), and the
plain PyTorch fp32 reference of the position-causal GQA attention
(reference model.py:110-129 restricted to rows S)."""
from __future__ import annotations

import numpy as np
import torch


def build_case(R=2, n=1000, H=8, G=2, frac=0.6, seed=0, layers=2, layer=1, device="cuda",
               scale_kv=1.0, scale_q=1.0, rope_theta=None):
    import paper_2503_16525_b200 as K
    from paper_2503_16525_b200.engine import Engine, RowSet
    from paper_2503_16525_b200.pool import CachePool, KVArena
    extra = {} if rope_theta is None else {"rope_theta": rope_theta}
    cfg = K.ModelConfig(num_layers=layers, num_heads=H, num_kv_heads=G, d_model=H * 128,
                        vocab_size=100, max_positions=n + 64, **extra)
    model = K.ToyModel(cfg, init="device")
    pages = R * ((n + 63) // 64)
    arena = KVArena(cfg, pages + 2)
    eng = Engine(model, CachePool(cfg, arena=arena))
    gen = torch.Generator(device=device).manual_seed(seed)
    st = eng.new_batch([np.zeros(n, dtype=np.int64) for _ in range(R)])
    arena.data.copy_((torch.randn(arena.data.shape, generator=gen, device=device) * scale_kv)
                     .to(torch.bfloat16))
    rng = np.random.default_rng(seed)
    req, pos, off = [], [], [0]
    for r in range(R):
        if frac >= 1.0:
            p = np.arange(n)
        else:
            p = np.sort(rng.choice(n, size=max(1, int(frac * n)), replace=False))
            if p[-1] != n - 1:
                p = np.append(p, n - 1)
        req.append(np.full(len(p), r, dtype=np.int32))
        pos.append(p.astype(np.int32))
        off.append(off[-1] + len(p))
    req, pos = np.concatenate(req), np.concatenate(pos)
    m = len(pos)
    rows = RowSet(m, torch.arange(m, dtype=torch.int32, device=device),
                  torch.from_numpy(req).to(device), torch.from_numpy(pos).to(device), None,
                  np.array(off, dtype=np.int64)).build_tiles(device, kv_len=[n] * R,
                                                             partial_first=frac < 1.0)
    q = (torch.randn(m, H, 128, generator=gen, device=device) * scale_q).to(torch.bfloat16)
    return eng, st, rows, q, layer


def reference(eng, st, rows, q, layer, heads=None):
    """fp32 torch attention of rows S over each request's paged K/V."""
    arena = eng.arena.data                          # [pages, L, 2, 64, G, 128]
    H, G = q.shape[1], arena.shape[4]
    heads = range(H) if heads is None else heads
    bt = st.block_table.cpu().numpy()
    out = torch.zeros(q.shape[0], len(heads), 128, device=q.device)
    for r in range(len(st.lengths)):
        a, b = int(rows.row_off[r]), int(rows.row_off[r + 1])
        if a == b:
            continue
        pos = rows.row_pos[a:b].long()
        kmax = int(pos.max()) + 1
        pg = torch.from_numpy(bt[r, :(kmax + 63) // 64].astype(np.int64)).to(q.device)
        kv = arena[pg, layer].float()                   # [p, 2, 64, G, 128]
        k = kv[:, 0].reshape(-1, G, 128)[:kmax]
        v = kv[:, 1].reshape(-1, G, 128)[:kmax]
        mask = torch.arange(kmax, device=q.device)[None, :] <= pos[:, None]
        for j, h in enumerate(heads):
            g = h // (H // G)
            s = (q[a:b, h].float() @ k[:, g].T) / np.sqrt(128.0)
            s = s.masked_fill(~mask, float("-inf"))
            out[a:b, j] = torch.softmax(s, dim=-1) @ v[:, g]
    return out


def attention_flops(rows, H):
    """Algorithmic FLOPs: sum over rows of 4*H*d*(p+1)."""
    return float((rows.row_pos.double() + 1).sum().item()) * 4 * H * 128
