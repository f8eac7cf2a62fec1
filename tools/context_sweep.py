"""Context-length sweep (BASELINE configs[4] at one GPU, 50% chunk hit): DHD
prefill throughput and batch latency of the Llama-3.1-8B-shape step for
requests of 2k..64k tokens, next to full recompute on the same GPU.  The
batch shrinks as the context grows (about 32k prompt tokens per step).

    python tools/context_sweep.py [--hit 0.5] [--steps 3] [--warmup 2] [--seqs 2048,4096]
                                  [--out profiles/x.json]
"""
import argparse
import gc
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2503_16525_b200.workload import request_batches  # noqa: E402

CONFIGS = [(2048, 16, 16), (4096, 8, 16), (8192, 4, 8), (16384, 2, 4), (32768, 1, 2),
           (65536, 1, 2)]      # (tokens per request, requests per step, pool sources)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--hit", type=float, default=0.5)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--seqs", default=None, help="comma-separated request lengths to run")
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--max-seq", type=int, default=65536)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    rows = []
    for seq, batch, sources in CONFIGS:
        if seq > a.max_seq or (a.seqs and str(seq) not in a.seqs.split(",")):
            continue
        args = argparse.Namespace(layers=a.layers, sources=sources, seq=seq, batch=batch)
        cfg, model, pool, eng, srcs = bench.build_engine(args, dev)
        batches = request_batches(srcs, a.steps + a.warmup, batch, seq, a.hit, cfg.vocab_size,
                                  seed=11)
        toks = [torch.from_numpy(np.concatenate(b)).to(dev) for b in batches]
        res = {"seq": seq, "batch": batch}
        for mode in ("selective", "full"):
            for i in range(a.warmup):
                eng.release(eng.prefill_batch(batches[i], ratio=0.2, mode=mode, tokens_dev=toks[i]))
            torch.cuda.synchronize()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps + 1)]
            ev[0].record()
            hits = []
            for k, i in enumerate(range(a.warmup, a.warmup + a.steps)):
                st = eng.prefill_batch(batches[i], ratio=0.2, mode=mode, tokens_dev=toks[i])
                hits.append(st.n_hit_dev.sum())
                eng.release(st)
                ev[k + 1].record()
            torch.cuda.synchronize()
            ms = ev[0].elapsed_time(ev[-1]) / a.steps
            res[mode] = {"ms_per_batch": ms, "tok_s": batch * seq / (ms / 1000.0),
                         "ms_each": [round(ev[k].elapsed_time(ev[k + 1]), 2)
                                     for k in range(a.steps)]}
            if mode == "selective":
                res["measured_hit"] = float(torch.stack(hits).double().mean().item()) / (batch * seq)
        res["dhd_speedup"] = res["full"]["ms_per_batch"] / res["selective"]["ms_per_batch"]
        rows.append(res)
        print(json.dumps(res), flush=True)
        del cfg, model, pool, eng, srcs, toks, batches
        gc.collect()
        torch.cuda.empty_cache()
    out = {"workload": f"llama3.1-8b-shape DHD prefill, {a.hit:.0%} chunk hit, r=0.2, "
                       f"{a.layers} layers, one B200", "rows": rows}
    if a.out:
        with open(a.out, "w") as fh:
            json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
