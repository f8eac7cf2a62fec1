"""A1 attention in isolation (diagnostic; run under gpurun).

    python tools/micro_attn.py [--reqs 8] [--seq 4096] [--frac 0.6] [--iters 20]

Times kvs_attention_fwd (variant from KVS_ATTN) over a DHD-like row set
(frac of each request's positions, scattered) with CUDA events, reports
TFLOP/s over the algorithmic FLOPs and checks two heads against the fp32
torch reference.
"""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from attn_case import attention_flops, build_case, reference  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reqs", type=int, default=8)
    ap.add_argument("--seq", type=int, default=4096)
    ap.add_argument("--frac", type=float, default=0.6)
    ap.add_argument("--heads", type=int, default=32)
    ap.add_argument("--kv", type=int, default=8)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--check", action="store_true")
    a = ap.parse_args()
    eng, st, rows, q, layer = build_case(a.reqs, a.seq, a.heads, a.kv, a.frac, seed=1)
    o = torch.empty_like(q)
    eng._attention(q, rows, layer, eng.arena.c, st.batch_c, o)
    torch.cuda.synchronize()
    if a.check:
        want = reference(eng, st, rows, q, layer, [0, a.heads - 1])
        err = ((o[:, [0, a.heads - 1]].float() - want).norm() / want.norm()).item()
        print(f"rel err vs fp32 torch: {err:.2e}")
    fl = attention_flops(rows, a.heads)
    ts = []
    for it in range(a.iters + 3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        eng._attention(q, rows, layer, eng.arena.c, st.batch_c, o)
        e1.record()
        torch.cuda.synchronize()
        if it >= 3:
            ts.append(e0.elapsed_time(e1))
    t = float(np.median(ts))
    print(f"variant={os.environ.get('KVS_ATTN', '3')} reqs={a.reqs} seq={a.seq} frac={a.frac} "
          f"rows={rows.n_rows} tiles={rows.n_tiles}: {t:.3f} ms  {fl / t / 1e9:.0f} TFLOP/s")


if __name__ == "__main__":
    main()
