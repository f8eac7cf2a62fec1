"""GPU idle-gap trace of bench steps (diagnostic; run under gpurun).

    python tools/step_trace.py [--steps 2] [bench args...]

Runs the bench engine (same workload as bench.py) under torch.profiler for a
few steps after warm-up and prints: device busy time per step, every GPU idle
gap longer than 20 us with the host-side call that was running when the gap
began, and the top kernels.  Writes gpurun_out/step_trace.json (chrome trace).
"""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    sys.argv = [sys.argv[0]] + [a for a in sys.argv[1:]]
    args = bench.parse()
    import numpy as np
    import torch
    from torch.profiler import ProfilerActivity, profile

    from paper_2503_16525_b200.workload import request_batches
    device = torch.device("cuda", 0)
    torch.cuda.set_device(device)
    cfg, model, pool, eng, sources = bench.build_engine(args, device)
    n = args.warmup + args.steps
    batches = request_batches(sources, n, args.batch, args.seq, args.hit, cfg.vocab_size, seed=1)
    toks = [torch.from_numpy(np.concatenate(b)).to(device) for b in batches]
    for i in range(args.warmup):
        eng.release(eng.prefill_batch(batches[i], ratio=args.ratio, tokens_dev=toks[i]))
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA], with_stack=True) as prof:
        for i in range(args.warmup, n):
            st = eng.prefill_batch(batches[i], ratio=args.ratio, tokens_dev=toks[i])
            eng.release(st)
        torch.cuda.synchronize()
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    path = os.path.join(ROOT, "gpurun_out", "step_trace.json")
    prof.export_chrome_trace(path)
    ev = json.load(open(path))["traceEvents"]
    gpu = sorted([e for e in ev if e.get("cat") == "kernel" or e.get("cat") == "gpu_memcpy"
                  or e.get("cat") == "gpu_memset"], key=lambda e: e["ts"])
    cpu = [e for e in ev if e.get("cat") in ("python_function", "cpu_op", "cuda_runtime")
           and "dur" in e]
    t0, t1 = gpu[0]["ts"], gpu[-1]["ts"] + gpu[-1]["dur"]
    busy = 0.0
    gaps = []
    end = gpu[0]["ts"]
    for e in gpu:
        if e["ts"] > end + 20:
            gaps.append((end, e["ts"] - end, e["name"]))
        busy += e["dur"]
        end = max(end, e["ts"] + e["dur"])
    print(f"span {(t1 - t0) / 1000:.2f} ms  kernel busy {busy / 1000:.2f} ms  "
          f"idle gaps>20us: {len(gaps)} totalling {sum(g[1] for g in gaps) / 1000:.2f} ms")
    py = [e for e in cpu if e.get("cat") == "python_function"]
    rt = [e for e in cpu if e.get("cat") == "cuda_runtime"]
    for ts, dur, nxt in sorted(gaps, key=lambda g: -g[1])[:25]:
        # host frames active when the gap started (innermost repo frames)
        act = [e["name"] for e in py if e["ts"] <= ts <= e["ts"] + e["dur"]
               and ("paper_2503" in e["name"] or "bench" in e["name"])]
        r = [e["name"] for e in rt if e["ts"] <= ts + dur and e["ts"] + e["dur"] >= ts]
        print(f"  gap {dur:8.1f} us before {nxt[:50]:50s} | runtime {r[:2]} | host {act[-3:]}")
    agg = {}
    for e in gpu:
        agg.setdefault(e["name"][:70], [0, 0.0])
        agg[e["name"][:70]][0] += 1
        agg[e["name"][:70]][1] += e["dur"]
    for k, (c, d) in sorted(agg.items(), key=lambda x: -x[1][1])[:25]:
        print(f"  {d / 1000 / args.steps:8.3f} ms/step {c // args.steps:4d}x  {k}")


if __name__ == "__main__":
    main()
