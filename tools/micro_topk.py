"""kvs_topk_select in isolation (diagnostic; run under gpurun): the one-CTA-
per-request top-B used by D2's selectors and by the F4 strategies.

    python tools/micro_topk.py [--reqs 8] [--seq 4096] [--frac 0.35] [--ratio 0.2]
"""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2503_16525_b200 import _native as N  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reqs", type=int, default=8)
    ap.add_argument("--seq", type=int, default=4096)
    ap.add_argument("--frac", type=float, default=0.35)
    ap.add_argument("--ratio", type=float, default=0.2)
    ap.add_argument("--iters", type=int, default=20)
    a = ap.parse_args()
    N.load()
    dev = torch.device("cuda")
    n = a.reqs * a.seq
    g = torch.Generator(device=dev).manual_seed(0)
    scores = torch.rand(n, device=dev, generator=g) * 900
    cand = torch.where(torch.rand(n, device=dev, generator=g) < a.frac, 0, -1).to(torch.int32)
    off = torch.arange(0, n + 1, a.seq, device=dev, dtype=torch.int64)
    nr = (cand.view(a.reqs, a.seq) >= 0).sum(1)
    bud = torch.ceil(nr.double() * a.ratio).to(torch.int32)
    sel = torch.zeros(n, dtype=torch.uint8, device=dev)
    args = (scores.data_ptr(), cand.data_ptr(), off.data_ptr(), a.reqs, a.seq, bud.data_ptr(),
            sel.data_ptr(), N.stream_ptr())
    N.call("kvs_topk_select", *args)
    torch.cuda.synchronize()
    # check
    s_np, c_np, sel_np = scores.cpu().numpy(), cand.cpu().numpy(), sel.cpu().numpy()
    ok = True
    for r in range(a.reqs):
        sl = slice(r * a.seq, (r + 1) * a.seq)
        idx = np.nonzero(c_np[sl] >= 0)[0]
        order = sorted(idx, key=lambda i: (-s_np[sl][i], i))[:int(bud[r])]
        want = np.zeros(a.seq, np.uint8)
        want[order] = 1
        ok &= bool((want == sel_np[sl]).all())
    ts = []
    for _ in range(a.iters):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        N.call("kvs_topk_select", *args)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"topk reqs={a.reqs} seq={a.seq} exact={ok}: median {np.median(ts) * 1e3:.1f} us")


if __name__ == "__main__":
    main()
