"""Library comparison point for A1 (diagnostic; run under gpurun): flashinfer's
sm100 cutlass FMHA on a full-causal ragged batch of the same shape micro_attn
times (8 x 4096 tokens, 32 query / 8 KV heads, head dim 128, bf16).  The
module is JIT-compiled on first use (minutes).

    python tools/fi_attn.py [--reqs 8] [--seq 4096] [--backend cutlass]
"""
import argparse

import torch


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reqs", type=int, default=8)
    ap.add_argument("--seq", type=int, default=4096)
    ap.add_argument("--heads", type=int, default=32)
    ap.add_argument("--kv", type=int, default=8)
    ap.add_argument("--backend", default="cutlass")
    ap.add_argument("--iters", type=int, default=20)
    a = ap.parse_args()
    import flashinfer
    dev = torch.device("cuda")
    n = a.reqs * a.seq
    q = torch.randn(n, a.heads, 128, device=dev, dtype=torch.bfloat16)
    k = torch.randn(n, a.kv, 128, device=dev, dtype=torch.bfloat16)
    v = torch.randn(n, a.kv, 128, device=dev, dtype=torch.bfloat16)
    indptr = torch.arange(0, n + 1, a.seq, device=dev, dtype=torch.int32)
    ws = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    w = flashinfer.prefill.BatchPrefillWithRaggedKVCacheWrapper(ws, "NHD", backend=a.backend)
    w.plan(indptr, indptr, a.heads, a.kv, 128, causal=True, q_data_type=torch.bfloat16)
    o = w.run(q, k, v)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.iters):
        o = w.run(q, k, v)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.iters
    flops = 4.0 * a.reqs * a.heads * 128 * (a.seq * (a.seq + 1) / 2)
    print(f"flashinfer[{a.backend}] reqs={a.reqs} seq={a.seq}: {ms:.3f} ms "
          f"{flops / ms / 1e9:.0f} TFLOP/s")
    # spot check one head against torch sdpa
    r = 0
    sl = slice(r * a.seq, (r + 1) * a.seq)
    qh = q[sl, 0].float()[None, None]
    kh = k[sl, 0].float()[None, None]
    vh = v[sl, 0].float()[None, None]
    ref = torch.nn.functional.scaled_dot_product_attention(qh, kh, vh, is_causal=True)[0, 0]
    err = ((o[sl, 0].float() - ref).norm() / ref.norm()).item()
    print(f"rel err head 0: {err:.2e}")


if __name__ == "__main__":
    main()
