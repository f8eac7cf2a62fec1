"""Multi-tenant serving stream (BASELINE configs[3] on one GPU): 256
Yi-1.5-9B-shape requests of 4096 tokens arrive over time with a bimodal hit
mix (half copy ~80% of their tokens from the shared sources, half ~20%; the
pattern of reference trace.py:115-150), the cache-aware scheduler
(scheduling.py:106-125) or FCFS forms batches, every batch runs through
Engine.prefill_batch on the GPU and is charged its measured device time
(serving.run_serving, reference simulate.py:140-215).  Completed requests are
written back zero-copy and the pool evicts LRU entries beyond its byte budget.

    python tools/serve_stream.py [--requests 256] [--batch 16] [--out profiles/x.json]
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
from paper_2503_16525_b200.serving import TraceRecord, run_serving  # noqa: E402
from paper_2503_16525_b200.workload import target_request  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--requests", type=int, default=256)
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--seq", type=int, default=4096)
    ap.add_argument("--gap-ms", type=float, default=4.0)
    ap.add_argument("--capacity-gb", type=float, default=48.0)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    import paper_2503_16525_b200 as K
    from paper_2503_16525_b200.pool import KVArena
    shape = dict(K.YI15_9B)
    page_bytes = KVArena.bytes_per_page(K.ModelConfig(**shape, max_positions=a.seq + 64))
    extra = int(a.capacity_gb * (1 << 30)) // page_bytes + 4 * a.batch * ((a.seq + 63) // 64)
    args = argparse.Namespace(layers=None, sources=16, seq=a.seq, batch=a.batch, shape="yi",
                              extra_pages=extra)
    cfg, model, pool, eng, sources = bench.build_engine(args, dev)
    rng = np.random.default_rng(3)
    trace = []
    for i in range(a.requests):
        hit = 0.8 if i % 2 == 0 else 0.2
        toks = target_request(sources, a.seq, hit, cfg.vocab_size, rng)
        trace.append(TraceRecord(f"q{i:04d}", round(i * a.gap_ms, 6), toks.tolist(), 0))
    out = {"workload": f"yi1.5-9b-shape serving stream: {a.requests} requests x {a.seq} tokens, "
                       f"bimodal hit 0.8/0.2, arrivals every {a.gap_ms} ms, batches of {a.batch}, "
                       f"r=0.2, pool budget {a.capacity_gb} GB (LRU), one B200",
           "runs": {}}
    for sched in ("cache_aware", "fcfs"):
        pool.capacity_bytes = int(a.capacity_gb * (1 << 30))
        rep = run_serving(trace, eng, batch_size=a.batch, ratio=0.2, scheduler=sched)
        agg = dict(rep.aggregate)
        ms = [b[2] for b in rep.batches]
        agg["batches"] = len(rep.batches)
        agg["measured_batch_ms_mean"] = float(np.mean(ms))
        agg["prefill_tok_s_device"] = a.requests * a.seq / (sum(ms) / 1000.0)
        out["runs"][sched] = agg
        print(sched, json.dumps(agg), flush=True)
        # drop the written-back requests so the second scheduler starts from
        # the same pool of sources
        for rid in [r.id for r in rep.requests]:
            if rid in pool.entries:
                pool._drop(pool.entries[rid])
    if a.out:
        with open(a.out, "w") as fh:
            json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
