"""Few-row attention (kvs_decode_attention: the tensor-core flash-decoding
kernel behind decode steps, probe queries and session recomputes) against a
plain PyTorch fp32 reference of the same op (reference engine.py:104-109 /
model.py:110-129 for the given rows): decode-step row sets (chosen rows plus
the new token of each request, sharing one chunk), probe queries (one row per
request: several requests per chunk), requests with more rows than a chunk,
GQA groups 1-8, single-key contexts and non-causal kv_len."""
import numpy as np
import pytest
import torch

from attn_case import build_case, reference

pytestmark = pytest.mark.gpu

TOL = 1e-2        # bf16 output of a bf16-operand / fp32-accumulate kernel


def _rows(eng, R, n, per_req, rng, device="cuda"):
    from paper_2503_16525_b200.engine import RowSet
    req, pos, off = [], [], [0]
    for r in range(R):
        k = per_req[r % len(per_req)]
        p = np.sort(rng.choice(n, size=min(k, n), replace=False)).astype(np.int32)
        if k >= 1 and p[-1] != n - 1:
            p[-1] = n - 1                              # the newest row sees the whole context
            p = np.unique(p)
        req.append(np.full(len(p), r, dtype=np.int32))
        pos.append(p)
        off.append(off[-1] + len(p))
    req, pos = np.concatenate(req), np.concatenate(pos)
    m = len(pos)
    return RowSet(m, torch.arange(m, dtype=torch.int32, device=device),
                  torch.from_numpy(req).to(device), torch.from_numpy(pos).to(device), None,
                  np.array(off, dtype=np.int64))


def _run(eng, st, rows, q, layer):
    o = torch.empty_like(q)
    eng._decode_attention(q, rows, layer, eng.arena.c, st.batch_c, o, int(st.capacity.max()))
    torch.cuda.synchronize()
    return o


@pytest.mark.parametrize("R,n,H,G,per_req", [
    (8, 4096, 32, 8, [4]),          # decode step: 3 chosen rows + the new token per request
    (8, 4096, 32, 8, [1]),          # probe queries: one row per request, 4 requests per chunk
    (3, 1000, 28, 4, [2, 5, 1]),    # Qwen group 7: two rows per chunk, runs across chunks
    (2, 700, 8, 1, [17, 3]),        # MHA: 16 rows per chunk, a request longer than a chunk
    (4, 129, 16, 2, [4, 9]),        # group 8
    (5, 1, 8, 4, [1]),              # single-key contexts
    (2, 3000, 12, 4, [6]),          # group 3 (15 of 16 M rows)
])
def test_decode_attention_vs_torch_fp32(R, n, H, G, per_req):
    rng = np.random.default_rng(n + H + R)
    eng, st, _, _, layer = build_case(R, n, H, G, 1.0, seed=n + G)
    rows = _rows(eng, R, n, per_req, rng)
    q = (torch.randn(rows.n_rows, H, 128, device="cuda") * 0.5).to(torch.bfloat16)
    got = _run(eng, st, rows, q, layer)
    want = reference(eng, st, rows, q, layer)
    err = (got.float() - want).norm() / want.norm()
    assert err < TOL, f"relative Frobenius error {err:.3e}"


def test_decode_attention_large_logits():
    """Peaked scores with the max growing across pages and splits."""
    rng = np.random.default_rng(1)
    eng, st, _, _, layer = build_case(2, 2500, 8, 2, 1.0, seed=4, scale_kv=3.0)
    rows = _rows(eng, 2, 2500, [4], rng)
    q = (torch.randn(rows.n_rows, 8, 128, device="cuda") * 4.0).to(torch.bfloat16)
    got = _run(eng, st, rows, q, layer)
    want = reference(eng, st, rows, q, layer)
    assert torch.isfinite(got).all()
    err = (got.float() - want).norm() / want.norm()
    assert err < TOL, f"relative Frobenius error {err:.3e}"
