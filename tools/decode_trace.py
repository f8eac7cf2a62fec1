"""Profile decode-stage DHD steps (diagnostic; run under gpurun).

    python tools/decode_trace.py [bench args]

Prefills one bench batch with decode capacity, runs decode steps under
torch.profiler, prints per-kernel device time per token step and the share
of idle GPU time (host-bound launches / syncs)."""
import json
import os
import sys

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2503_16525_b200.workload import request_batches  # noqa: E402


def main():
    args = bench.parse()
    dev = torch.device("cuda", 0)
    cfg, model, pool, eng, sources = bench.build_engine(args, dev)
    batch = request_batches(sources, 1, args.batch, args.seq, args.hit, cfg.vocab_size, seed=1)[0]
    st = eng.prefill_batch(batch, ratio=args.ratio, decode_capacity=8)
    rng = np.random.default_rng(0)
    eng.decode_step(st, rng.integers(0, cfg.vocab_size, len(batch)), 3)
    torch.cuda.synchronize()
    steps = 3
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        for _ in range(steps):
            tok = torch.from_numpy(rng.integers(0, cfg.vocab_size, len(batch))).to(dev)
            eng.decode_step_device(st, tok, 3)
        torch.cuda.synchronize()
    path = os.path.join(ROOT, "gpurun_out", "decode_trace.json")
    os.makedirs(os.path.dirname(path), exist_ok=True)
    prof.export_chrome_trace(path)
    ev = json.load(open(path))["traceEvents"]
    gpu = sorted([e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")],
                 key=lambda e: e["ts"])
    span = (gpu[-1]["ts"] + gpu[-1]["dur"] - gpu[0]["ts"]) / 1000
    busy = sum(e["dur"] for e in gpu) / 1000
    print(f"{steps} decode steps: span {span:.2f} ms, kernel busy {busy:.2f} ms")
    agg = {}
    for e in gpu:
        k = e["name"][:70]
        agg.setdefault(k, [0, 0.0])
        agg[k][0] += 1
        agg[k][1] += e["dur"]
    for k, (c, d) in sorted(agg.items(), key=lambda x: -x[1][1])[:20]:
        print(f"  {d / 1000 / steps:8.3f} ms/step {c // steps:4d}x  {k}")


if __name__ == "__main__":
    main()
