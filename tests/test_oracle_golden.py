"""Pin the CPU oracle against golden vectors produced by the reference itself.

The oracle (oracle/) is test infrastructure; these tests make it trustworthy
as the parity checker for the CUDA path.
"""
import numpy as np
import pytest

from golden_io import MODEL_CASES, match_doc, model_case, reuse_of, weights_digest
from oracle import kvshare_oracle as O

DOC = match_doc()


def test_window_hashes_golden():
    for case in DOC["hashes"]:
        got = O.window_hashes(case["tokens"], case["w"], case["b"], case["m"])
        assert [int(x) for x in got] == case["hashes"]


def test_known_answer_hash():
    assert [int(x) for x in O.window_hashes([1, 2, 3], 3)] == [1026]  # test_matching.py:45-48


@pytest.mark.parametrize("idx", range(len(DOC["match"])))
def test_match_pairs_golden(idx):
    c = DOC["match"][idx]
    tm, cm = O.match_pairs(c["target"], c["candidate"], c["w"], c["b"], c["m"])
    assert tm == c["tm"] and cm == c["cm"]


@pytest.mark.parametrize("idx", range(len(DOC["lookup"])))
def test_pool_lookup_golden(idx):
    c = DOC["lookup"][idx]
    se, sc, contrib = O.pool_lookup(c["entries_newest_first"], c["request"], c["w"], c["b"], c["m"])
    pos = np.nonzero(se >= 0)[0].tolist()
    assert pos == c["positions"]
    assert se[pos].tolist() == c["src_entry"]
    assert sc[pos].tolist() == c["src_cand"]
    ids = c["entry_ids_newest_first"]
    assert sorted(ids[i] for i in np.nonzero(contrib)[0]) == sorted(c["contributors_lru_order"])


def test_schedule_golden():
    for c in DOC["schedule"]:
        got = O.schedule_order(c["hit"], c["arrival"], c["ids"], c["batch_size"], c["aging"], c["now"])
        assert [[c["ids"][i] for i in b] for b in got] == c["batches"]


@pytest.mark.parametrize("name", MODEL_CASES)
def test_weights_draw_golden(name):
    cfg, z = model_case(name)
    W = O.draw_weights(cfg)
    assert weights_digest(W) == str(z["weights_sha256"])


@pytest.mark.parametrize("name", MODEL_CASES)
def test_probe_scores_selection_golden(name):
    cfg, z = model_case(name)
    W = O.draw_weights(cfg)
    reuse = reuse_of(z)
    probe = 1 if cfg.num_layers >= 2 else 0
    q, kt, vt, kp, vp = O.perturbed_probe(z["target"], W, cfg, reuse, probe)
    for a, b in ((q, "probe_q"), (kt, "probe_k_true"), (vt, "probe_v_true"),
                 (kp, "probe_k_pert"), (vp, "probe_v_pert")):
        np.testing.assert_allclose(a, z[b], rtol=0, atol=1e-12)
    states, selected, eligible, info = O.prefill_with_selection(
        z["target"], W, cfg, reuse, float(z["ratio"]))
    np.testing.assert_allclose(info["scores"], z["scores"], rtol=1e-12, atol=1e-14)
    assert tuple(selected) == tuple(z["selected"].tolist())
    assert sorted(eligible) == z["eligible"].tolist()
    np.testing.assert_allclose(states["hidden"], z["prefill_hidden"], atol=1e-12)
    np.testing.assert_allclose(states["k"], z["prefill_k"], atol=1e-12)
    np.testing.assert_allclose(states["v"], z["prefill_v"], atol=1e-12)


@pytest.mark.parametrize("name", MODEL_CASES)
def test_partial_rows_prefill_equals_reference(name):
    """computing only the query rows
    S = non-reused U selected U {n-1} (O.forward_rows, the restatement the
    large parity tests use) reproduces the reference's own prefill states on
    rows S, and its K/V caches are the reference's complete caches."""
    cfg, z = model_case(name)
    W = O.draw_weights(cfg)
    reuse = reuse_of(z)
    n = len(z["target"])
    sel = z["selected"].tolist()
    got = O.forward_rows(z["target"], W, cfg, reuse, sel)
    S = got["rows"]
    assert S.tolist() == sorted((set(range(n)) - set(reuse.reused)) | set(sel) | {n - 1})
    assert len(S) < n
    np.testing.assert_allclose(got["hidden"], z["prefill_hidden"][:, S], rtol=0, atol=1e-12)
    np.testing.assert_allclose(got["k"], z["prefill_k"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(got["v"], z["prefill_v"], rtol=0, atol=1e-12)
    with pytest.raises(ValueError):              # a fresh row outside the computed set
        O.forward_rows(z["target"], W, cfg, reuse, sel, rows=S[1:] if S[0] not in
                       set(reuse.reused) else S[:-1])


@pytest.mark.parametrize("kvh,rope", [(None, None), (2, 10000.0)])
def test_per_head_restatement_equals_batched(kvh, rope, monkeypatch):
    """The one-head-at-a-time attention / alpha used above O._BIG equals the
    batched (H, n, n) restatement, and forward_rows equals forward on rows S
    with GQA and RoPE."""
    cfg = O.OracleConfig(3, 4, 64, 300, 3, kvh, rope)
    W = O.draw_weights(cfg)
    table = O.rope_table(512, cfg.d_k, rope) if rope else None
    rng = np.random.default_rng(0)
    q = rng.normal(size=(4, 97, 16))
    k = rng.normal(size=(cfg.kvh, 97, 16))
    v = rng.normal(size=(cfg.kvh, 97, 16))
    want, _ = O.attention(q, k, v, causal=True, group=cfg.group)
    want_a = O.dhd_alpha(q, k, group=cfg.group)
    monkeypatch.setattr(O, "_BIG", 0)
    got, attn = O.attention(q, k, v, causal=True, group=cfg.group)
    assert attn is None
    np.testing.assert_allclose(got, want, rtol=0, atol=1e-13)
    np.testing.assert_allclose(O.dhd_alpha(q, k, group=cfg.group), want_a, rtol=0, atol=1e-13)
    toks = rng.integers(0, 300, 60)
    src = toks[10:40]
    st = O.forward(src, W, cfg, table=table)
    se = np.full(60, -1, np.int32)
    sc = np.full(60, -1, np.int32)
    se[10:40], sc[10:40] = 0, np.arange(30)
    reuse = O.Reuse(se, sc, [st["k"]], [st["v"]])
    sel = [12, 30, 39]
    full = O.forward(toks, W, cfg, reuse, {l: set(sel) for l in range(3)}, table)
    part = O.forward_rows(toks, W, cfg, reuse, sel, table=table)
    S = part["rows"]
    np.testing.assert_allclose(part["hidden"], full["hidden"][:, S], rtol=0, atol=1e-12)
    np.testing.assert_allclose(part["k"], full["k"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(part["v"], full["v"], rtol=0, atol=1e-12)


@pytest.mark.parametrize("name", MODEL_CASES)
def test_decode_golden(name):
    cfg, z = model_case(name)
    W = O.draw_weights(cfg)
    reuse = reuse_of(z)
    states, selected, eligible, _ = O.prefill_with_selection(
        z["target"], W, cfg, reuse, float(z["ratio"]))
    sess = O.Session(z["target"], W, cfg, states, reuse.reused, selected)
    q_t0 = sess.query_rows_probe(int(z["decode_tokens"][0]))
    np.testing.assert_allclose(q_t0, z["decode_q_t0"], atol=1e-12)
    chosen0, scores0 = O.select_decode_step(q_t0, sess.k[sess.probe_layer], sess.delta_v_probe(),
                                           eligible, int(z["n_extra"]))
    np.testing.assert_allclose(scores0, z["decode_scores0"], atol=1e-13)
    assert tuple(chosen0) == tuple(z["decode_chosen0"].tolist())
    chosen, _ = O.run_generation(sess, z["decode_tokens"], int(z["n_extra"]), eligible)
    assert [len(c) for c in chosen] == z["decode_recompute_counts"].tolist()
    assert [list(c) for c in chosen if c] == [c.tolist() for c in z["decode_chosen"]]
    np.testing.assert_allclose(sess.k, z["final_k"], atol=1e-12)
    np.testing.assert_allclose(sess.v, z["final_v"], atol=1e-12)


def test_budget_exact_double_ceil():
    assert O.budget(0.55, 100) == 56           # SURVEY finding 6
    assert O.budget(0.3, 10) == 3 and O.budget(0.01, 7) == 1 and O.budget(1.0, 7) == 7


def test_known_answer_selection():
    # test_selection.py:36-43 - uniform attention picks the largest deviation
    rng = np.random.default_rng(0)
    k = rng.normal(size=(3, 8))
    dv = np.zeros((3, 8))
    dv[0, 0], dv[1, 0], dv[2, 0] = 0.5, 0.2, 0.9
    sel, _ = O.select_prefill(np.zeros((3, 8)), k, dv, {0, 1, 2}, 1 / 3, causal=False)
    assert sel == (2,)
    # test_selection.py:95-108 - decode concentration
    n, d = 8, 4
    k = np.full((n, d), -1.0)
    k[5] = [12.0, 0.0, 0.0, 0.0]
    sel, _ = O.select_decode_step(np.array([4.0, 0, 0, 0]), k, np.ones((n, d)), set(range(n)), 1)
    assert sel == (5,)


def _fixed_doc():
    import json
    import os
    return json.load(open(os.path.join(os.path.dirname(__file__), "golden",
                                       "golden_fixed_chunk.json")))


@pytest.mark.parametrize("idx", range(40))
def test_fixed_chunk_lookup_golden(idx):
    """F5 restatement pinned to the reference's own fixed-chunk lookups."""
    c = _fixed_doc()[idx]
    se, sc, contrib = O.fixed_chunk_lookup(c["entries_newest_first"], c["request"], c["chunk"])
    pos = np.nonzero(se >= 0)[0].tolist()
    assert pos == c["positions"]
    assert se[pos].tolist() == c["src_entry"]
    assert sc[pos].tolist() == c["src_cand"]
    ids = c["entry_ids_newest_first"]
    assert sorted(ids[i] for i in np.nonzero(contrib)[0]) == sorted(c["contributors_lru_order"])


def _strategies():
    import os
    return np.load(os.path.join(os.path.dirname(__file__), "golden", "golden_strategies.npz"))


@pytest.mark.parametrize("strategy", ["magnitude", "positional", "random", "ideal",
                                      "attention_weighted"])
def test_select_baseline_golden(strategy):
    """F4 restatement pinned to the reference's select_baseline outputs."""
    z = _strategies()
    for c in range(int(z["n_cases"])):
        g = lambda k: z[f"c{c}_{k}"]  # noqa: E731
        ratio, seed = g("meta")
        idx, scores = O.select_baseline(strategy, g("q"), g("k"), g("v"), g("dk"), g("dv"),
                                        g("reused").tolist(), float(ratio), int(seed))
        assert list(idx) == g(f"{strategy}_idx").tolist()
        np.testing.assert_allclose(scores, g(f"{strategy}_scores"), rtol=1e-9, atol=1e-12)


def _oracle_mode_case():
    import os
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden_oracle_mode.npz"))
    L, H, d_model, vocab, seed = (int(x) for x in z["config"])
    ocfg = O.OracleConfig(L, H, d_model, vocab, seed)
    W = O.draw_weights(ocfg)
    E = int(z["n_entries"])
    reuse = O.Reuse(z["src_entry"], z["src_cand"], [z[f"entry_k_{i}"] for i in range(E)],
                    [z[f"entry_v_{i}"] for i in range(E)])
    return z, ocfg, W, reuse


@pytest.mark.parametrize("strategy", ["magnitude", "positional", "random", "ideal",
                                      "attention_weighted"])
def test_oracle_mode_prefill_golden(strategy):
    """ORACLE-mode restatement (engine.py:245-285) pinned to the reference run."""
    z, ocfg, W, reuse = _oracle_mode_case()
    ref = {"k": z["ref_k"], "v": z["ref_v"]}
    sets, hidden = O.oracle_prefill(z["target"], W, ocfg, reuse, strategy, 0.3, ref, seed=5)
    for layer, st in enumerate(sets):
        assert sorted(st) == z[f"{strategy}_set{layer}"].tolist()
    np.testing.assert_allclose(hidden, z[f"{strategy}_hidden"], rtol=1e-9, atol=1e-9)
