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
