"""Drop-in session API through the GPU path, replaying the reference's own
runs (tests/golden/golden_model_*.npz, written by tests/golden/make_golden.py
from the compiled reference):

* ``ReuseSession(model, tokens, reuse, recompute)`` prefill K/V (engine.py:47-75);
* ``.query_rows_probe`` (engine.py:150-171) against the golden q_t of step 0;
* ``.delta_v_probe`` (engine.py:140-148) through the step-0 decode scores;
* ``.recompute_positions`` + ``.append`` (engine.py:114-138) along the
  reference's recorded decode trajectory, ending at its final K/V;
* ``run_generation`` (engine.py:298-328): recompute counts, chosen positions
  and per-step deviations against the oracle, which is pinned to the same
  goldens (tests/test_oracle_golden.py).
"""
import numpy as np
import pytest

from golden_io import MODEL_CASES, model_case, reuse_of
from oracle import kvshare_oracle as O
from parity import assert_rel_fro, assert_scores_close, assert_selection_tie_band

pytestmark = pytest.mark.gpu


def _golden_pool(z, cfg):
    import paper_2503_16525_b200 as K
    from paper_2503_16525_b200.pool import CachePool
    kcfg = K.ModelConfig(cfg.num_layers, cfg.num_heads, cfg.d_model, cfg.vocab_size, cfg.seed)
    model = K.init_model(kcfg)
    pool = CachePool(kcfg, K.HashParams(window_size=int(z["w"])), arena_pages=64)
    E = len(z["entry_tokens"])
    for i in reversed(range(E)):                      # golden order is newest first
        pool.insert(f"src{E - 1 - i}", z["entry_tokens"][i], z["entry_k"][i], z["entry_v"][i])
    reuse = pool.lookup(z["target"])
    assert sorted(reuse.sources) == np.nonzero(z["src_entry"] >= 0)[0].tolist()
    return K, model, pool, reuse


def _trajectory(z):
    """The reference run_generation's recompute_positions calls per step."""
    log = iter([c.tolist() for c in z["decode_chosen"]])
    return [next(log) if c else [] for c in z["decode_recompute_counts"].tolist()]


@pytest.mark.parametrize("name", MODEL_CASES)
def test_session_methods_replay_reference(name):
    cfg, z = model_case(name)
    K, model, pool, reuse = _golden_pool(z, cfg)
    selected = set(z["selected"].tolist())
    sess = K.ReuseSession(model, z["target"], reuse, recompute=selected)
    assert_rel_fro(sess.k, z["prefill_k"], 3e-2)
    assert_rel_fro(sess.v, z["prefill_v"], 3e-2)
    # step 0: probe query and the decode-stage scores built from delta_v_probe
    toks = z["decode_tokens"].tolist()
    q_t0 = sess.query_rows_probe(toks[0])
    assert_rel_fro(q_t0, z["decode_q_t0"], 3e-2)
    eligible = set(z["eligible"].tolist())
    dv = sess.delta_v_probe()
    assert dv.shape == (cfg.num_heads, sess.n_tokens, cfg.d_k)
    res0 = K.select_decode_step(q_t0, sess.k[sess.probe_layer], dv, eligible, int(z["n_extra"]))
    assert_scores_close(res0.scores, z["decode_scores0"], 2e-2)
    assert_selection_tie_band(res0.indices, z["decode_chosen0"].tolist(), z["decode_scores0"],
                              len(z["decode_chosen0"]), 2e-2)
    # the reference's decode trajectory through recompute_positions + append
    W = O.draw_weights(cfg)
    ostates, _, _, _ = O.prefill_with_selection(z["target"], W, cfg, reuse_of(z),
                                                float(z["ratio"]))
    osess = O.Session(z["target"], W, cfg, ostates, reuse_of(z).reused, selected)
    for tok, chosen in zip(toks, _trajectory(z)):
        if chosen:
            sess.recompute_positions(chosen)
            osess.recompute_positions(chosen)
            assert set(chosen) <= set(sess.recomputed[0])
        out = sess.append(tok)
        want = osess.append(tok)
        assert_rel_fro(out.hidden_out, want, 3e-2)
    assert sess.n_tokens == len(z["target"]) + len(toks)
    assert_rel_fro(sess.k, z["final_k"], 3e-2)
    assert_rel_fro(sess.v, z["final_v"], 3e-2)


@pytest.mark.parametrize("name", MODEL_CASES)
def test_run_generation_vs_reference(name):
    cfg, z = model_case(name)
    K, model, pool, reuse = _golden_pool(z, cfg)
    ratio, n_extra = float(z["ratio"]), int(z["n_extra"])
    res = K.prefill_with_selection(model, z["target"], reuse, K.SelectionConfig(ratio=ratio))
    ref = K.ReuseSession(model, z["target"])
    toks = z["decode_tokens"].tolist()
    gen = K.run_generation(res.session, ref, toks, n_extra)
    assert gen.recompute_counts == z["decode_recompute_counts"].tolist()
    # oracle twin of the same run, following the GPU's own prefill selection
    W = O.draw_weights(cfg)
    oreuse = reuse_of(z)
    sel = set(res.selected)
    ost = O.forward(z["target"], W, cfg, oreuse, {l: sel for l in range(cfg.num_layers)})
    osess = O.Session(z["target"], W, cfg, ost, oreuse.reused, sel)
    oref = O.Session(z["target"], W, cfg, O.forward(z["target"], W, cfg))
    eligible = set(oreuse.reused) - sel
    want_dev, hmax = [], 1.0
    for tok, got in zip(toks, gen.chosen):
        want, scores = O.select_decode_step(osess.query_rows_probe(tok),
                                            osess.k[osess.probe_layer], osess.delta_v_probe(),
                                            eligible, n_extra)
        assert_selection_tie_band(got, want, scores, len(want), 2e-2)
        osess.recompute_positions(got)
        eligible -= set(got)
        h = osess.append(tok)
        want_dev.append(np.linalg.norm(h - oref.append(tok)))
        hmax = max(hmax, np.linalg.norm(h))
    if tuple(res.selected) == tuple(z["selected"].tolist()) and \
            [list(c) for c in gen.chosen if c] == [c.tolist() for c in z["decode_chosen"]]:
        assert_rel_fro(res.session.k, z["final_k"], 3e-2)
        assert_rel_fro(res.session.v, z["final_v"], 3e-2)
    np.testing.assert_allclose(gen.step_deviation, want_dev, rtol=0.1, atol=2e-2 * hmax)
    assert gen.cumulative_deviation == pytest.approx(sum(gen.step_deviation))


def test_stale_reuse_map_raises_and_sessions_release_pages():
    """A ReuseMap whose entry was evicted or replaced must not gather from
    the slot's next owner (CacheError); sessions return their arena pages
    when dropped, so a loop of sessions on one pool does not exhaust it."""
    import gc

    import paper_2503_16525_b200 as K
    from paper_2503_16525_b200.pool import CachePool
    cfg = K.ModelConfig(num_layers=2, num_heads=2, d_model=32, vocab_size=256, seed=3)
    model = K.init_model(cfg)
    pool = CachePool(cfg, K.HashParams(window_size=4), arena_pages=24)
    rng = np.random.default_rng(0)
    src = rng.integers(0, 256, 120)
    st = O.forward(src, O.draw_weights(O.OracleConfig(2, 2, 32, 256, 3)), O.OracleConfig(
        2, 2, 32, 256, 3))
    pool.insert("a", src, st["k"], st["v"])
    target = np.concatenate([rng.integers(0, 256, 10), src[5:90]])
    free0 = pool.arena.free_pages
    for _ in range(40):                        # 40 sessions x 6 pages >> 24-page arena
        sess = K.ReuseSession(model, target, pool.lookup(target), decode_capacity=256)
        sess.append(7)
        del sess
        gc.collect()
    assert pool.arena.free_pages == free0
    reuse = pool.lookup(target)
    pool.insert("a", src[::-1].copy(), st["k"][:, :, ::-1], st["v"][:, :, ::-1])   # replaces "a"
    with pytest.raises(K.CacheError):
        K.ReuseSession(model, target, reuse)
    with pytest.raises(K.CacheError):
        next(iter(reuse.sources.values()))[0].k
