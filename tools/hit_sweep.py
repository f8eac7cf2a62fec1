"""Hit-rate sweep (BASELINE configs[4] at one GPU; SURVEY F2's concave-latency
premise): DHD prefill throughput and batch latency of the Llama-3.1-8B-shape
step for chunk hit rates 0..0.9, next to full recompute on the same GPU.

    python tools/hit_sweep.py [--seq 4096] [--batch 8] [--steps 3] [--warmup 2] [--out profiles/x.json]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2503_16525_b200.scheduling import LatencyModel  # noqa: E402
from paper_2503_16525_b200.workload import request_batches  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seq", type=int, default=4096)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    args = argparse.Namespace(layers=a.layers, sources=16, seq=a.seq, batch=a.batch)
    dev = torch.device("cuda", 0)
    cfg, model, pool, eng, sources = bench.build_engine(args, dev)
    rows = []
    for mode, hit in [("full", 0.0)] + [("selective", h) for h in np.arange(0.0, 0.95, 0.1)]:
        batches = request_batches(sources, a.steps + a.warmup, a.batch, a.seq, float(hit),
                                  cfg.vocab_size, seed=11)
        toks = [torch.from_numpy(np.concatenate(b)).to(dev) for b in batches]
        for i in range(a.warmup):
            eng.release(eng.prefill_batch(batches[i], ratio=0.2, mode=mode, tokens_dev=toks[i]))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        hits = []
        for i in range(a.warmup, a.warmup + a.steps):
            st = eng.prefill_batch(batches[i], ratio=0.2, mode=mode, tokens_dev=toks[i])
            hits.append(st.n_hit_dev.sum())
            eng.release(st)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.steps
        h = float(torch.stack(hits).double().mean().item()) / (a.batch * a.seq)
        rows.append({"mode": mode, "target_hit": round(float(hit), 2), "measured_hit": h,
                     "ms_per_batch": ms, "tok_s": a.batch * a.seq / (ms / 1000.0)})
        print(json.dumps(rows[-1]), flush=True)
    sel = [r for r in rows if r["mode"] == "selective"]
    f = np.array([r["ms_per_batch"] for r in sel])
    hs = np.array([r["measured_hit"] for r in sel])
    decreasing = bool(np.all(np.diff(f) <= 1e-6 * f[0] + 0.02 * f[0]))
    # concavity on the measured grid: second differences <= 0 (within 2 % noise)
    second = f[:-2] - 2 * f[1:-1] + f[2:]
    concave = bool(np.all(second <= 0.02 * f[0]))
    doc = {"workload": f"llama3.1-8b shape, {a.batch} x {a.seq} tokens, L={a.layers}, r=0.2",
           "rows": rows, "decreasing": decreasing, "concave_within_2pct": concave,
           "reference_latency_model": {"t_base_ms": LatencyModel().t_base_ms,
                                       "t_comp_ms": LatencyModel().t_comp_ms,
                                       "exponent": LatencyModel().exponent},
           "hit_grid": hs.tolist()}
    print(json.dumps({k: doc[k] for k in ("decreasing", "concave_within_2pct")}))
    if a.out:
        with open(a.out, "w") as fh:
            json.dump(doc, fh, indent=1)


if __name__ == "__main__":
    main()
