"""Per-step jitter of the DHD prefill step: device time per step (CUDA events) next
to the host time spent inside prefill_batch, with the Python garbage collector
on and off, to find occasional slow steps.

    python tools/step_jitter.py [--seq 2048] [--batch 16] [--steps 20]
"""
import argparse
import gc
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2503_16525_b200.workload import request_batches  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seq", type=int, default=2048)
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--layers", type=int, default=32)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    args = argparse.Namespace(layers=a.layers, sources=16, seq=a.seq, batch=a.batch)
    cfg, model, pool, eng, srcs = bench.build_engine(args, dev)
    n = 2 + 2 * a.steps
    batches = request_batches(srcs, n, a.batch, a.seq, 0.5, cfg.vocab_size, seed=11)
    toks = [torch.from_numpy(np.concatenate(b)).to(dev) for b in batches]
    for i in range(2):
        eng.release(eng.prefill_batch(batches[i], ratio=0.2, mode="selective", tokens_dev=toks[i]))
    torch.cuda.synchronize()
    for label, gc_on in (("gc_on", True), ("gc_off", False)):
        (gc.enable if gc_on else gc.disable)()
        base = 2 + (0 if gc_on else a.steps)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps + 1)]
        host = []
        ev[0].record()
        for k in range(a.steps):
            i = base + k
            t0 = time.perf_counter()
            st = eng.prefill_batch(batches[i], ratio=0.2, mode="selective", tokens_dev=toks[i])
            eng.release(st)
            host.append(round((time.perf_counter() - t0) * 1e3, 2))
            ev[k + 1].record()
        torch.cuda.synchronize()
        dev_ms = [round(ev[k].elapsed_time(ev[k + 1]), 2) for k in range(a.steps)]
        print(json.dumps({"mode": label, "device_ms": dev_ms, "host_ms": host,
                          "gc_counts": gc.get_count()}), flush=True)
    gc.enable()


if __name__ == "__main__":
    main()
