"""D1 DHD-alpha in isolation (diagnostic; run under gpurun).

    python tools/micro_alpha.py [--reqs 8] [--seq 4096] [--heads 32] [--kv 8] [--iters 20]

Times kvs_dhd_alpha (pass 1 row LSE + pass 2 key-major column sums + the
kv-head reduce) over full-causal probe tiles of R requests with CUDA events,
reports TFLOP/s over the algorithmic FLOPs 2*H*d*n(n+1) per request (SURVEY.md
8d) and checks alpha of two requests against an fp32 torch restatement."""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from attn_case import build_case  # noqa: E402


def torch_alpha(eng, st, q, layer, r, H, G):
    arena = eng.arena.data
    bt = st.block_table.cpu().numpy()
    n = int(st.lengths[r])
    a = int(st.req_off_host[r])
    pg = torch.from_numpy(bt[r, :(n + 63) // 64].astype(np.int64)).to(q.device)
    k = arena[pg, layer, 0].float().reshape(-1, G, 128)[:n]
    mask = torch.ones(n, n, dtype=torch.bool, device=q.device).tril()
    al = torch.zeros(n, device=q.device)
    for h in range(H):
        s = (q[a:a + n, h].float() @ k[:, h // (H // G)].T) / np.sqrt(128.0)
        al += torch.softmax(s.masked_fill(~mask, float("-inf")), dim=-1).sum(0)
    return al / H


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reqs", type=int, default=8)
    ap.add_argument("--seq", type=int, default=4096)
    ap.add_argument("--heads", type=int, default=32)
    ap.add_argument("--kv", type=int, default=8)
    ap.add_argument("--iters", type=int, default=20)
    a = ap.parse_args()
    from paper_2503_16525_b200 import _native as N
    eng, st, rows, q, layer = build_case(R=a.reqs, n=a.seq, H=a.heads, G=a.kv, frac=1.0)
    H, G = a.heads, a.kv
    n_tot = rows.n_rows
    alpha = torch.empty(n_tot, dtype=torch.float32, device="cuda")
    ws = torch.empty(N.ws_bytes("kvs_dhd_alpha_workspace", n_tot, H, G), dtype=torch.uint8,
                     device="cuda")
    lse = torch.empty(n_tot, H, dtype=torch.float32, device="cuda")

    def run_alpha():
        N.call("kvs_dhd_alpha", q.data_ptr(), H, 1, layer, eng.arena.c, st.batch_c,
               rows.row_pos.data_ptr(), rows.tiles[0].data_ptr(), rows.tiles[1].data_ptr(),
               rows.tiles[2].data_ptr(), rows.n_tiles, None, eng.scale, alpha.data_ptr(),
               ws.data_ptr(), ws.numel(), N.stream_ptr())

    def run_pass1():
        N.call("kvs_attention_fwd", q.data_ptr(), rows.row_pos.data_ptr(), n_tot, H,
               rows.tiles[0].data_ptr(), rows.tiles[1].data_ptr(), rows.tiles[2].data_ptr(),
               rows.n_tiles, None, 1, layer, eng.arena.c, st.batch_c, eng.scale, None,
               lse.data_ptr(), N.stream_ptr())

    flops = sum(2.0 * H * 128 * l * (l + 1) for l in st.lengths)
    out = {"reqs": a.reqs, "seq": a.seq, "heads": H, "kv_heads": G}
    for name, fn, fl in (("alpha", run_alpha, flops), ("pass1_lse", run_pass1, flops / 2)):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.iters
        out[name] = {"ms": ms, "tflops": fl / ms / 1e9}
    out["pass2_colsum_ms_est"] = out["alpha"]["ms"] - out["pass1_lse"]["ms"]
    run_alpha()
    err = 0.0
    for r in range(min(2, a.reqs)):
        want = torch_alpha(eng, st, q, layer, r, H, G)
        got = alpha[int(st.req_off_host[r]):int(st.req_off_host[r + 1])]
        err = max(err, float(((got - want).abs().max() / want.abs().max()).item()))
    out["max_rel_err_vs_torch"] = err
    import json
    print(json.dumps(out))


if __name__ == "__main__":
    main()
