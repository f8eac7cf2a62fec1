"""D2 DHD-select in isolation (diagnostic; run under gpurun).

    python tools/micro_select.py [--reqs 8] [--seq 4096] [--hit 0.5] [--iters 50]

Builds a Llama-shape arena (kv_heads 8, head_dim 128, 32 layers), v_true and
alpha for a batch of requests with reused spans, then times kvs_dhd_select
with CUDA events (L2 flushed between launches) and checks dv-L1, scores and
the selected set against torch / numpy.  Prints achieved GB/s over the
algorithmic bytes (2*G*d*2 + 12 B per reused row + 4 B per
selected row).
"""
from __future__ import annotations

import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2503_16525_b200 as K  # noqa: E402
from paper_2503_16525_b200 import _native as N  # noqa: E402
from paper_2503_16525_b200.engine import Engine  # noqa: E402
from paper_2503_16525_b200.pool import CachePool, KVArena  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reqs", type=int, default=8)
    ap.add_argument("--seq", type=int, default=4096)
    ap.add_argument("--hit", type=float, default=0.5)
    ap.add_argument("--ratio", type=float, default=0.2)
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--profile", action="store_true")
    ap.add_argument("--nosel", action="store_true", help="budget 0: streaming phase only")
    ap.add_argument("--trace-csv", default=None)
    ap.add_argument("--trace", action="store_true",
                    help="library built with -DKVS_SEL_TRACE (KVS_LIB): per-CTA phase timeline")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    shape = dict(K.LLAMA31_8B)
    shape["num_layers"] = a.layers
    shape["vocab_size"] = 1000
    cfg = K.ModelConfig(**shape, max_positions=a.seq + 64)
    model = K.ToyModel(cfg, init="device")
    pages = a.reqs * ((a.seq + 63) // 64)
    arena = KVArena(cfg, pages + 4)
    eng = Engine(model, CachePool(cfg, arena=arena))
    rng = np.random.default_rng(0)
    st = eng.new_batch([rng.integers(0, 1000, a.seq) for _ in range(a.reqs)])
    arena.data.normal_()
    n = a.reqs * a.seq
    G, d = cfg.kv_heads, 128
    # reused spans of 64..1024 tokens covering ~hit of every request
    src = np.full(n, -1, dtype=np.int32)
    for r in range(a.reqs):
        p = 0
        while p < a.seq:
            span = int(rng.integers(64, 1025))
            if rng.random() < a.hit:
                src[r * a.seq + p: r * a.seq + min(a.seq, p + span)] = 0
            p += span
    st.src_slot = torch.from_numpy(src).to(dev)
    v_true = (torch.randn(n, G, d, device=dev) * 0.5).to(torch.bfloat16)
    alpha = torch.rand(n, device=dev)
    n_hit = np.array([(src[r * a.seq:(r + 1) * a.seq] >= 0).sum() for r in range(a.reqs)])
    bud = np.array([K.SelectionConfig(ratio=a.ratio).budget(int(h)) for h in n_hit], np.int32)
    if a.nosel:
        bud[:] = 0
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    layer = 1
    dv, score, sel = eng._select(st, v_true, alpha, bud)
    torch.cuda.synchronize()
    # ---- check
    vc = arena.data[:, layer, 1]                      # [pages, 64, G, d]
    bt = st.block_table.cpu().numpy()
    pos = np.arange(n) % a.seq
    req = np.arange(n) // a.seq
    pg = torch.from_numpy(bt[req, pos // 64].astype(np.int64)).to(dev)
    rows = vc[pg, torch.from_numpy(pos % 64).to(dev)]        # [n, G, d]
    want_dv = (rows.float() - v_true.float()).abs().sum(dim=(1, 2))
    want_dv[torch.from_numpy(src < 0).to(dev)] = 0
    err = ((dv - want_dv).abs().max() / want_dv.abs().max()).item()
    sc = (alpha * want_dv).cpu().numpy()
    got_sel = sel.cpu().numpy().astype(bool)
    ok = True
    for r in range(a.reqs):
        sl = slice(r * a.seq, (r + 1) * a.seq)
        reused = np.nonzero(src[sl] >= 0)[0]
        s_dev = score.cpu().numpy()[sl]
        order = sorted(reused, key=lambda i: (-s_dev[i], i))[:bud[r]]
        want = np.zeros(a.seq, bool)
        want[order] = True
        ok &= bool((want == got_sel[sl]).all())
    print(f"dv-L1 rel err {err:.2e}; selection exact vs device scores: {ok}; "
          f"score err {np.abs(score.cpu().numpy() - sc).max() / sc.max():.2e}")
    # ---- timing
    nbytes = n_hit.sum() * (2 * G * d * 2 + 12) + 4 * bud.sum()
    # direct C-ABI launches on preallocated buffers (no host work between the events)
    bud_dev = torch.from_numpy(bud).to(dev)
    ws = eng._ws["select"].get(N.ws_bytes("kvs_dhd_select_workspace", n, a.reqs), dev, zero=True)
    args = (v_true.data_ptr(), alpha.data_ptr(), st.src_slot.data_ptr(), layer, eng.arena.c,
            st.batch_c, bud_dev.data_ptr(), dv.data_ptr(), score.data_ptr(), sel.data_ptr(),
            ws.data_ptr(), ws.numel(), N.stream_ptr())
    ts = []
    for it in range(a.iters + 3):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        N.call("kvs_dhd_select", *args)
        e1.record()
        torch.cuda.synchronize()
        if it >= 3:
            ts.append(e0.elapsed_time(e1))
    t = float(np.median(ts))
    if a.trace:
        import ctypes
        lib = N.load()
        lib.kvs_sel_trace_dump.restype = ctypes.c_int32
        buf = np.zeros(1024 * 8, dtype=np.uint64)
        lib.kvs_sel_trace_dump(buf.ctypes.data, buf.size)        # clear
        flush.zero_()
        torch.cuda.synchronize()
        N.call("kvs_dhd_select", *args)
        torch.cuda.synchronize()
        lib.kvs_sel_trace_dump(buf.ctypes.data, buf.size)
        tr = buf.reshape(1024, 8)[:148].astype(np.int64)
        t0 = tr[:, 0].min()
        names = ["start", "meta", "streamed", "sel_start", "sel_end", "keys", "radix", "pass0"]
        for ph in (1, 2, 3, 5, 7, 6, 4):
            v = tr[:, ph]
            v = v[v > 0] - t0
            if len(v):
                print(f"  {names[ph]:>9}: min {v.min() / 1e3:6.2f} med {np.median(v) / 1e3:6.2f} "
                      f"max {v.max() / 1e3:6.2f} us (n={len(v)})")
        st0 = tr[:, 0] - t0
        if a.trace_csv:
            np.savetxt(a.trace_csv, tr - t0, fmt="%d", delimiter=",")
        print(f"  start spread: max {st0.max() / 1e3:.2f} us")
    print(f"reqs={a.reqs} seq={a.seq} reused={n_hit.sum()} bytes={nbytes / 1e6:.1f} MB  "
          f"median {t * 1e3:.1f} us  min {min(ts) * 1e3:.1f} us  -> {nbytes / t / 1e6:.0f} GB/s")


if __name__ == "__main__":
    main()
