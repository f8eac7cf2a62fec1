"""D1/D2/D3 parity on the GPU against the fp64 oracle on bf16-rounded inputs,
plus the reference's known-answer selection tests."""
import math

import numpy as np
import pytest

from oracle import kvshare_oracle as O
from parity import assert_scores_close, assert_selection_tie_band, bf16

pytestmark = pytest.mark.gpu


def _rand(rng, shape, scale=1.0):
    return bf16(rng.normal(size=shape) * scale)


@pytest.mark.parametrize("H,G,n,d,causal", [
    (1, 1, 5, 4, True), (2, 2, 37, 8, True), (4, 4, 130, 16, True), (4, 2, 300, 64, True),
    (8, 2, 257, 128, True), (2, 1, 129, 32, False), (4, 4, 64, 128, False),
    (32, 8, 512, 128, True)])
def test_v_impact_scores_vs_oracle(H, G, n, d, causal):
    from paper_2503_16525_b200.deviation import alpha_scores
    rng = np.random.default_rng(H * 1000 + n)
    q = _rand(rng, (H, n, d))
    k = _rand(rng, (G, n, d))
    dv = _rand(rng, (G, n, d), 0.1)
    scores, dv_l1, alpha, _ = alpha_scores(q, k, dv, causal)
    want_alpha = O.dhd_alpha(q, k, causal=causal, group=H // G)
    want = O.v_impact_scores(q, k, dv, causal=causal, group=H // G)
    assert_scores_close(alpha, want_alpha, 5e-3)
    np.testing.assert_allclose(dv_l1, np.abs(dv).sum(axis=(0, 2)), rtol=1e-5)
    assert_scores_close(scores, want)


def test_alpha_sums_to_row_count():
    """Column sums of a row-stochastic causal matrix add up to n per head."""
    from paper_2503_16525_b200.deviation import alpha_scores
    rng = np.random.default_rng(5)
    q, k = _rand(rng, (4, 1000, 128)), _rand(rng, (4, 1000, 128))
    _, _, alpha, _ = alpha_scores(q, k, np.zeros_like(k), True)
    assert abs(alpha.sum() - 1000) < 1000 * 2e-3


@pytest.mark.parametrize("seed", range(4))
def test_select_prefill_vs_oracle(seed):
    import paper_2503_16525_b200 as K
    rng = np.random.default_rng(seed)
    H, G, n, d = 4, 2, int(rng.integers(50, 400)), 64
    q, k, dv = _rand(rng, (H, n, d)), _rand(rng, (G, n, d)), _rand(rng, (G, n, d), 0.1)
    reused = sorted(rng.choice(n, size=int(rng.integers(1, n)), replace=False).tolist())
    dv[:, [i for i in range(n) if i not in set(reused)]] = 0
    ratio = float(rng.choice([0.1, 0.2, 0.3, 0.55, 1.0]))
    res = K.select_prefill(q, k, dv, reused, K.SelectionConfig(ratio=ratio))
    want, scores = O.select_prefill(q, k, dv, reused, ratio, group=H // G)
    assert len(res.indices) == O.budget(ratio, len(reused))
    assert list(res.indices) == sorted(res.indices)
    assert_selection_tie_band(res.indices, want, scores, O.budget(ratio, len(reused)))
    assert_scores_close(res.scores, scores)


def test_select_prefill_known_answers():
    import paper_2503_16525_b200 as K
    rng = np.random.default_rng(0)
    k = rng.normal(size=(3, 8))
    dv = np.zeros((3, 8))
    dv[0, 0], dv[1, 0], dv[2, 0] = 0.5, 0.2, 0.9
    res = K.select_prefill(np.zeros((3, 8)), k, dv, {0, 1, 2}, K.SelectionConfig(ratio=1 / 3),
                           causal=False)
    assert res.indices == (2,)                                   # test_selection.py:36-43
    q, kk = rng.normal(size=(2, 5, 4))
    res = K.select_prefill(q, kk, np.zeros((5, 4)), {0, 1, 2, 3, 4}, K.SelectionConfig(ratio=0.4))
    assert res.indices == (0, 1)                                 # ties break low
    res = K.select_prefill(q, kk, rng.normal(size=(5, 4)), {1, 2, 4}, K.SelectionConfig(ratio=1.0))
    assert res.indices == (1, 2, 4)
    with pytest.raises(K.ParameterError):
        K.select_prefill(q, kk, np.zeros((5, 4)), set(), K.SelectionConfig())
    assert K.SelectionConfig(ratio=0.55).budget(100) == 56


def test_select_decode_step_known_answers():
    import paper_2503_16525_b200 as K
    n, d = 8, 4
    k = np.full((n, d), -1.0)
    k[5] = [12.0, 0.0, 0.0, 0.0]
    q_t = np.array([4.0, 0.0, 0.0, 0.0])
    res = K.select_decode_step(q_t, k, np.ones((n, d)), set(range(n)), 1)
    assert res.indices == (5,)                                   # test_selection.py:95-108
    w = np.exp(q_t @ k.T / 2.0)
    w /= w.sum()
    np.testing.assert_allclose(res.scores, w * 4.0, atol=2e-3)
    rng = np.random.default_rng(1)
    k = rng.normal(size=(4, 8))
    assert K.select_decode_step(rng.normal(size=8), k, np.zeros((4, 8)), set(), 3).indices == ()
    assert K.select_decode_step(rng.normal(size=8), k, rng.normal(size=(4, 8)), {1, 3},
                                10).indices == (1, 3)
    assert K.select_decode_step(rng.normal(size=8), k, np.ones((4, 8)), {0, 1}, 0).indices == ()


@pytest.mark.parametrize("H,G,n", [(2, 2, 50), (4, 1, 333), (28, 4, 2000), (32, 8, 4096)])
def test_select_decode_step_vs_oracle(H, G, n):
    import paper_2503_16525_b200 as K
    rng = np.random.default_rng(n)
    q_t = _rand(rng, (H, 128), 0.3)
    k = _rand(rng, (G, n, 128))
    dv = _rand(rng, (G, n, 128), 0.1)
    elig = set(rng.choice(n, size=n // 3, replace=False).tolist())
    res = K.select_decode_step(q_t, k, dv, elig, 3)
    want, scores = O.select_decode_step(q_t, k, dv, elig, 3, group=H // G)
    assert_scores_close(res.scores, scores)
    assert_selection_tie_band(res.indices, want, scores, 3)


@pytest.mark.parametrize("n", [1000, 4096, 5000, 20000, 60000])
def test_select_exact_ties_large(n):
    """D2 top-B with massive exact score ties at sizes that take the register
    (<= 4096), shared-memory (<= 47104) and global key paths: uniform
    attention (q = 0, non-causal) makes every alpha identical, and dv rows
    drawn from three values make whole tie bands; the device must pick
    exactly the (-score, position) order of selection.py:63-66."""
    import paper_2503_16525_b200 as K
    rng = np.random.default_rng(n)
    d = 8
    q = np.zeros((1, n, d))
    k = _rand(rng, (1, n, d))
    dv = np.repeat(rng.choice([0.0, 0.5, 1.0], size=n)[None, :, None], d, axis=2)
    reused = sorted(rng.choice(n, size=n // 2, replace=False).tolist())
    cfg = K.SelectionConfig(ratio=0.3)
    res = K.select_prefill(q, k, dv, reused, cfg, causal=False)
    s = np.asarray(res.scores)
    want = sorted(sorted(reused, key=lambda i: (-s[i], i))[:cfg.budget(len(reused))])
    assert list(res.indices) == want
