"""A1 selective-recompute attention kernel (kvs_attention_fwd) against a
plain PyTorch fp32 reference of the same op (reference model.py:110-129 on
the rows S of a partial prefill), at Llama-like head shapes: full causal
prefill, scattered DHD row sets, GQA group sizes 1-8, ragged tails, and
adversarial score ranges that exercise the lazy O rescale."""
import pytest
import torch

from attn_case import build_case, reference

pytestmark = pytest.mark.gpu

# bf16 output of a bf16-operand / fp32-accumulate kernel vs fp32 reference
ATTN_TOL = 1e-2


def _run(eng, st, rows, q, layer):
    o = torch.empty_like(q)
    eng._attention(q, rows, layer, eng.arena.c, st.batch_c, o)
    torch.cuda.synchronize()
    return o


@pytest.mark.parametrize("R,n,H,G,frac", [
    (1, 1, 2, 1, 1.0), (1, 127, 2, 2, 1.0), (2, 129, 4, 2, 1.0), (1, 1000, 8, 2, 0.6),
    (3, 513, 8, 8, 0.3), (2, 2048, 32, 8, 0.6), (1, 4096, 32, 8, 1.0), (2, 777, 8, 1, 0.5),
    (1, 3000, 28, 4, 0.55)])
def test_attention_vs_torch_fp32(R, n, H, G, frac):
    eng, st, rows, q, layer = build_case(R, n, H, G, frac, seed=n + H)
    got = _run(eng, st, rows, q, layer)
    heads = sorted({0, H // 2, H - 1})
    want = reference(eng, st, rows, q, layer, heads)
    err = (got[:, heads].float() - want).norm() / want.norm()
    assert err < ATTN_TOL, f"relative Frobenius error {err:.3e}"


@pytest.mark.parametrize("scale_q", [4.0, 16.0])
def test_attention_large_logits_rescale(scale_q):
    """Peaked softmax with growing row maxima (lazy 2^8 rescale path)."""
    eng, st, rows, q, layer = build_case(1, 1500, 8, 2, 0.7, seed=3, scale_q=scale_q)
    got = _run(eng, st, rows, q, layer)
    want = reference(eng, st, rows, q, layer, [0, 5])
    err = (got[:, [0, 5]].float() - want).norm() / want.norm()
    assert err < ATTN_TOL, f"relative Frobenius error {err:.3e}"
    assert torch.isfinite(got).all()


@pytest.mark.parametrize("R,n,H,G,frac", [
    (2, 700, 8, 2, 0.6), (1, 1500, 28, 4, 0.55), (2, 300, 4, 4, 1.0), (1, 2048, 32, 8, 0.6),
    (3, 129, 8, 1, 0.5)])
def test_attention_qkv_fused_rope_bit_exact(R, n, H, G, frac):
    """kvs_attention_fwd_qkv (un-rotated q read from the projection rows and
    rotated in shared memory) equals the scatter-rotated q through
    kvs_attention_fwd bit for bit, for head pairs (fwd3) and single heads
    (fwd6); the scatter's K/V writes are identical with q_out == NULL."""
    eng, st, rows, _, layer = build_case(R, n, H, G, frac, seed=n + G, rope_theta=5e5)
    assert eng.rope_c is not None
    gen = torch.Generator(device="cuda").manual_seed(7)
    m = rows.n_rows
    qkv = (torch.randn(m, (H + 2 * G) * 128, generator=gen, device="cuda") * 2).to(torch.bfloat16)
    before = eng.arena.data.clone()
    q = torch.empty(m, H, 128, dtype=torch.bfloat16, device="cuda")
    eng._scatter(qkv, rows, layer, eng.arena.c, st.batch_c, q, use_write=False)
    want = _run(eng, st, rows, q, layer)
    arena_a = eng.arena.data.clone()
    eng.arena.data.copy_(before)
    eng._scatter(qkv, rows, layer, eng.arena.c, st.batch_c, None, use_write=False)
    torch.cuda.synchronize()
    assert torch.equal(eng.arena.data, arena_a), "scatter without q changed the K/V writes"
    got = torch.empty_like(want)
    eng._attention_qkv(qkv, rows, layer, eng.arena.c, st.batch_c, got)
    torch.cuda.synchronize()
    assert torch.equal(got, want), \
        f"fused-rope attention differs: max |d| {(got.float() - want.float()).abs().max():.3e}"
    ref = reference(eng, st, rows, q, layer, [0, H - 1])
    err = (got[:, [0, H - 1]].float() - ref).norm() / ref.norm()
    assert err < ATTN_TOL


@pytest.mark.parametrize("R,n,H,G,frac,one_shot", [
    (8, 1500, 32, 8, 0.6, "3"), (2, 3000, 28, 4, 0.55, "6"), (1, 300, 8, 1, 1.0, "6"),
    (1, 129, 2, 1, 1.0, "3")])
def test_persistent_kernels_match_one_shot(R, n, H, G, frac, one_shot, monkeypatch):
    """The persistent kernels (fwdp for even GQA groups, fwd6p for odd) walk
    ticketed (tile, head) items; each item's arithmetic is the one-shot
    kernel's (fwd3 / fwd6), so outputs are bit-identical, and a second launch
    (the ticket counter reset by the previous launch's last CTA) repeats them."""
    eng, st, rows, q, layer = build_case(R, n, H, G, frac, seed=R * n + G)
    monkeypatch.delenv("KVS_ATTN", raising=False)
    got = _run(eng, st, rows, q, layer)
    again = _run(eng, st, rows, q, layer)
    monkeypatch.setenv("KVS_ATTN", one_shot)
    want = _run(eng, st, rows, q, layer)
    assert torch.equal(got, again), "persistent kernel not deterministic across launches"
    assert torch.equal(got, want), \
        f"persistent vs one-shot: max |d| {(got.float() - want.float()).abs().max():.3e}"
