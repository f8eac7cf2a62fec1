"""A1 fixed per-CTA cost (diagnostic; run under gpurun).

    python tools/micro_attn_overhead.py

Full-causal row sets whose tiles all have the same key-block count are timed
for n_kb = 1, 2, 4, 8, 16 (sequence 128 * n_kb, requests chosen so every
launch has ~4 waves of CTAs).  A least-squares fit of time per CTA-wave
against n_kb separates the per-block cost from the fixed cost of a CTA
(prologue: TMEM alloc, barrier init, Q/K TMA latency, first Q.K^T;
epilogue: O read-back and store).  Each case is timed with q dense
(kvs_attention_fwd) and with q read un-rotated from QKV rows
(kvs_attention_fwd_qkv, rotation in shared memory).
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from attn_case import build_case  # noqa: E402
from paper_2503_16525_b200.engine import RowSet  # noqa: E402


def timed(fn, iters=20):
    ts = []
    for it in range(iters + 3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        if it >= 3:
            ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def main():
    H, G = 32, 8
    out = []
    for n_kb in (1, 2, 4, 8, 16):
        seq = 128 * n_kb
        # one tile per 128 rows; keep only each request's LAST tile so every
        # CTA sees n_kb key blocks: frac=1 rows, then restrict tiles
        reqs = max(1, (4 * 148 * 2) // (H // 2) // 1)       # 4 waves of head-pair CTAs
        eng, st, rows, q, layer = build_case(reqs, seq, H, G, 1.0, seed=n_kb, rope_theta=5e5)
        # tiles of the last 128 positions of each request only
        last0 = torch.tensor([int(rows.row_off[r + 1]) - 128 for r in range(reqs)],
                             dtype=torch.int32, device="cuda")
        treq = torch.arange(reqs, dtype=torch.int32, device="cuda")
        trows = torch.full((reqs,), 128, dtype=torch.int32, device="cuda")
        rows.tiles = torch.stack([treq, last0, trows]).contiguous()
        rows.n_tiles = reqs
        m = rows.n_rows
        qkv = torch.randn(m, (H + 2 * G) * 128, device="cuda").to(torch.bfloat16)
        o = torch.empty(m, H, 128, dtype=torch.bfloat16, device="cuda")
        t_dense = timed(lambda: eng._attention(q, rows, layer, eng.arena.c, st.batch_c, o))
        t_qkv = timed(lambda: eng._attention_qkv(qkv, rows, layer, eng.arena.c, st.batch_c, o))
        ctas = reqs * (H // 2)
        waves = ctas / 148.0
        out.append({"n_kb": n_kb, "ctas": ctas, "ms_dense": t_dense, "ms_qkv": t_qkv,
                    "us_per_wave_dense": 1e3 * t_dense / waves,
                    "us_per_wave_qkv": 1e3 * t_qkv / waves})
        print(json.dumps(out[-1]), flush=True)
    x = np.array([r["n_kb"] for r in out], dtype=np.float64)
    for key in ("dense", "qkv"):
        y = np.array([r[f"us_per_wave_{key}"] for r in out])
        b, a = np.polyfit(x, y, 1)
        print(json.dumps({"fit": key, "fixed_us_per_cta": a, "us_per_key_block": b}))


if __name__ == "__main__":
    main()
