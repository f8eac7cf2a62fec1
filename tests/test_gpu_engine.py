"""End-to-end parity of the device engine (A1 attention, G1 gather, probe,
partial prefill, decode-stage DHD) against the fp64 oracle run on the same
bf16-rounded weights; golden reference runs for the kvlab configs."""
import numpy as np
import pytest
import torch

from golden_io import MODEL_CASES, model_case
from oracle import kvshare_oracle as O
from parity import (HIDDEN_TOL, assert_rel_fro, assert_scores_close, assert_selection_tie_band,
                    bf16)

pytestmark = pytest.mark.gpu


def _models(L=3, H=2, d_model=16, vocab=256, seed=42, kvh=None, rope=None):
    import paper_2503_16525_b200 as K
    cfg = K.ModelConfig(num_layers=L, num_heads=H, d_model=d_model, vocab_size=vocab, seed=seed,
                        num_kv_heads=kvh, rope_theta=rope, max_positions=4096)
    model = K.init_model(cfg)
    emb, layers = model.host_weights
    W = {"embedding": bf16(emb), "layers": [tuple(bf16(w) for w in l) for l in layers]}
    ocfg = O.OracleConfig(L, H, d_model, vocab, seed, kvh, rope)
    table = O.rope_table(4096, cfg.d_k, rope) if rope else None
    return model, W, ocfg, table


@pytest.mark.parametrize("kw", [dict(), dict(L=2, H=4, d_model=256, kvh=2),
                                dict(L=2, H=4, d_model=512, kvh=1, rope=10000.0),
                                dict(L=3, H=8, d_model=1024, kvh=2, rope=500000.0)])
def test_model_forward_vs_oracle(kw):
    import paper_2503_16525_b200 as K
    model, W, ocfg, table = _models(**kw)
    rng = np.random.default_rng(0)
    for n in (1, 7, 130, 300):
        toks = rng.integers(0, ocfg.vocab_size, n)
        got = K.model_forward(toks, model)
        want = O.forward(toks, W, ocfg, table=table)
        assert_rel_fro(got.hidden, want["hidden"])
        assert_rel_fro(got.k, want["k"])
        assert_rel_fro(got.v, want["v"])
        assert_rel_fro(got.head_out, want["head_out"], 3e-2)


def _scenario(model, W, ocfg, table, rng, n_src=2, w=4):
    """Sources in the pool (oracle K/V so both sides see identical cached
    rows), target copying spans (studies._reuse_scenario pattern)."""
    import paper_2503_16525_b200 as K
    from paper_2503_16525_b200.pool import CachePool
    pool = CachePool(model.config, K.HashParams(window_size=w), arena_pages=256)
    srcs = []
    for s in range(n_src):
        src = rng.integers(0, ocfg.vocab_size, int(rng.integers(40, 90))).tolist()
        st = O.forward(src, W, ocfg, table=table)
        pool.insert(f"src{s}", src, bf16(st["k"]), bf16(st["v"]))
        srcs.append(src)
    target = rng.integers(0, ocfg.vocab_size, 5).tolist() + srcs[0][3:30] + \
        rng.integers(0, ocfg.vocab_size, 4).tolist() + srcs[-1][2:25] + \
        rng.integers(0, ocfg.vocab_size, 3).tolist()
    reuse = pool.lookup(target)
    order = sorted(pool.entries.values(), key=lambda e: -e.insert_seq)
    se, sc, _ = O.pool_lookup([e.tokens for e in order], target, w)
    ek = [e.k for e in order]
    ev = [e.v for e in order]
    oreuse = O.Reuse(se, sc, ek, ev)
    assert sorted(reuse.sources) == oreuse.reused
    return pool, target, reuse, oreuse


@pytest.mark.parametrize("kw", [dict(), dict(L=4, H=4, d_model=512, kvh=2, rope=10000.0),
                                dict(L=2, H=4, d_model=512)])
def test_gather_rows_exact_and_rope_aligned(kw):
    import paper_2503_16525_b200 as K
    model, W, ocfg, table = _models(**kw)
    rng = np.random.default_rng(1)
    pool, target, reuse, oreuse = _scenario(model, W, ocfg, table, rng)
    sess = K.ReuseSession(model, target, reuse)
    k = sess.k
    v = sess.v
    for layer in range(ocfg.num_layers):
        pos, kr, vr = oreuse.cached_rows(layer, table)
        np.testing.assert_array_equal(v[layer][:, pos], vr)       # V: bit-exact copy
        if table is None:
            np.testing.assert_array_equal(k[layer][:, pos], kr)   # K: bit-exact copy
        else:                                                      # K: re-aligned, <= 1 ulp
            np.testing.assert_allclose(k[layer][:, pos], bf16(kr), rtol=2 ** -7, atol=1e-6)
    if table is not None:
        # realigned layer-0 K equals fresh layer-0 K (context-free layer)
        fresh = O.forward(target, W, ocfg, table=table)["k"][0]
        pos = np.array(reuse.sources and sorted(reuse.sources))
        np.testing.assert_allclose(k[0][:, pos], fresh[:, pos], rtol=2 ** -6, atol=1e-4)


@pytest.mark.parametrize("kw,ratio", [(dict(), 0.3), (dict(L=4, H=4, d_model=512, kvh=2), 0.2),
                                      (dict(L=3, H=8, d_model=1024, kvh=2, rope=10000.0), 0.25)])
def test_prefill_with_selection_vs_oracle(kw, ratio):
    import paper_2503_16525_b200 as K
    model, W, ocfg, table = _models(**kw)
    rng = np.random.default_rng(2)
    pool, target, reuse, oreuse = _scenario(model, W, ocfg, table, rng)
    res = K.prefill_with_selection(model, target, reuse, K.SelectionConfig(ratio=ratio))
    states, want_sel, elig, info = O.prefill_with_selection(target, W, ocfg, oreuse, ratio, table)
    B = O.budget(ratio, len(oreuse.reused))
    assert_selection_tie_band(res.selected, want_sel, info["scores"], B)
    st = res.session.state
    assert_scores_close(st.score.double().cpu().numpy(), info["scores"])
    # forward parity on rows S with the GPU's own selection
    gpu_sel = set(res.selected)
    states = O.forward(target, W, ocfg, oreuse, {l: gpu_sel for l in range(ocfg.num_layers)},
                       table)
    n = len(target)
    S = sorted((set(range(n)) - set(oreuse.reused)) | gpu_sel | {n - 1})
    got = res.session.prefill_states
    assert np.isfinite(got.hidden[:, S]).all()
    assert_rel_fro(got.hidden[:, S], states["hidden"][:, S])
    assert_rel_fro(res.session.k, states["k"])
    assert_rel_fro(res.session.v, states["v"])
    assert res.eligible == set(oreuse.reused) - gpu_sel


@pytest.mark.parametrize("name", MODEL_CASES)
def test_prefill_golden_reference(name):
    """Reference kvlab run (golden): selected set, scores, prefill K/V."""
    import paper_2503_16525_b200 as K
    from paper_2503_16525_b200.pool import CachePool
    cfg, z = model_case(name)
    kcfg = K.ModelConfig(cfg.num_layers, cfg.num_heads, cfg.d_model, cfg.vocab_size, cfg.seed)
    model = K.init_model(kcfg)
    pool = CachePool(kcfg, K.HashParams(window_size=int(z["w"])), arena_pages=64)
    for i in reversed(range(len(z["entry_tokens"]))):
        pool.insert(f"src{len(z['entry_tokens']) - 1 - i}", z["entry_tokens"][i],
                    z["entry_k"][i], z["entry_v"][i])
    target = z["target"]
    reuse = pool.lookup(target)
    assert sorted(reuse.sources) == np.nonzero(z["src_entry"] >= 0)[0].tolist()
    res = K.prefill_with_selection(model, target, reuse, K.SelectionConfig(ratio=float(z["ratio"])))
    B = O.budget(float(z["ratio"]), len(reuse.sources))
    assert_selection_tie_band(res.selected, z["selected"], z["scores"], B)
    assert_scores_close(res.session.state.score.double().cpu().numpy(), z["scores"], 2e-2)
    if tuple(res.selected) == tuple(z["selected"].tolist()):
        assert_rel_fro(res.session.k, z["prefill_k"], 3e-2)
        assert_rel_fro(res.session.v, z["prefill_v"], 3e-2)
        n = len(target)
        S = sorted((set(range(n)) - set(reuse.sources)) | set(res.selected) | {n - 1})
        assert_rel_fro(res.session.prefill_states.hidden[:, S], z["prefill_hidden"][:, S], 3e-2)


@pytest.mark.parametrize("kw", [dict(), dict(L=3, H=4, d_model=512, kvh=2, rope=10000.0)])
def test_decode_stage_vs_oracle(kw):
    import paper_2503_16525_b200 as K
    model, W, ocfg, table = _models(**kw)
    rng = np.random.default_rng(3)
    pool, target, reuse, oreuse = _scenario(model, W, ocfg, table, rng)
    ratio = 0.2
    res = K.prefill_with_selection(model, target, reuse, K.SelectionConfig(ratio=ratio))
    gpu_sel = set(res.selected)
    states = O.forward(target, W, ocfg, oreuse, {l: gpu_sel for l in range(ocfg.num_layers)},
                       table)
    osess = O.Session(target, W, ocfg, states, oreuse.reused, gpu_sel, table)
    eligible = set(oreuse.reused) - gpu_sel
    sess = res.session
    eng, st = sess.engine, sess.state
    for step, tok in enumerate(rng.integers(0, ocfg.vocab_size, 8).tolist()):
        q_t = osess.query_rows_probe(tok)
        want, scores = O.select_decode_step(q_t, osess.k[osess.probe_layer],
                                            osess.delta_v_probe(), eligible, 3,
                                            group=ocfg.group)
        sess._grow(1)
        h, chosen = eng.decode_step(st, [tok], 3)
        sess.tokens.append(tok)
        assert_selection_tie_band(chosen[0], want, scores, len(want))
        osess.recompute_positions(chosen[0])
        eligible -= set(chosen[0])
        h_ref = osess.append(tok)
        assert_rel_fro(h[0].double().cpu().numpy(), h_ref, 3e-2)
    assert_rel_fro(sess.k, osess.k, 3e-2)


def test_run_generation_api():
    import paper_2503_16525_b200 as K
    model, W, ocfg, table = _models()
    rng = np.random.default_rng(4)
    pool, target, reuse, oreuse = _scenario(model, W, ocfg, table, rng)
    res = K.prefill_with_selection(model, target, reuse, K.SelectionConfig(ratio=0.2))
    ref = K.ReuseSession(model, target)
    gen = K.run_generation(res.session, ref, rng.integers(0, 256, 6).tolist(), 3)
    assert len(gen.step_deviation) == 6 and all(np.isfinite(gen.step_deviation))
    assert all(0 <= c <= 3 for c in gen.recompute_counts)
    # no reuse -> session equals the reference session
    plain = K.ReuseSession(model, target)
    ref2 = K.ReuseSession(model, target)
    gen2 = K.run_generation(plain, ref2, [1, 2, 3], 3)
    assert max(gen2.step_deviation) < 1e-3 and gen2.recompute_counts == [0, 0, 0]


@pytest.mark.parametrize("rope", [None, 10000.0])
def test_peer_gather_equals_local_gather(rope):
    """kvs_gather_kv_peer with every slot marked as owned by "rank 0" whose
    peer base is this process's own arena reads the same pages as the local
    G1: the destination K/V must be bit-identical (the peer-memory transport's
    kernel path, exercised without a second process)."""
    import torch

    from paper_2503_16525_b200 import _native as N
    kw = dict(L=3, H=4, d_model=512, kvh=2) if rope is None else \
        dict(L=3, H=4, d_model=512, kvh=2, rope=rope)
    model, W, ocfg, table = _models(**kw)
    rng = np.random.default_rng(5)
    pool, target, reuse, oreuse = _scenario(model, W, ocfg, table, rng)
    from paper_2503_16525_b200.engine import Engine
    eng = Engine(model, pool)
    st = eng.new_batch([np.asarray(target)])
    eng.lookup(st)
    assert int((st.src_slot >= 0).sum()) > 0
    idx = pool._build_index()
    eng.gather(st)
    want = eng.arena.data.clone()
    for p in st.pages[0]:
        eng.arena.data[p].zero_()
    owner = torch.zeros(idx["slot_pages"].shape[0], dtype=torch.int32, device=eng.device)
    base = torch.tensor([eng.arena.data.data_ptr()], dtype=torch.int64, device=eng.device)
    N.call("kvs_gather_kv_peer", eng.arena.c, st.batch_c, st.src_slot.data_ptr(),
           st.src_cand.data_ptr(), idx["slot_pages"].data_ptr(), idx["slot_max_pages"],
           owner.data_ptr(), base.data_ptr(), 0, ocfg.num_layers, eng._rope(), N.stream_ptr())
    torch.cuda.synchronize()
    hit_pos = (st.src_slot >= 0).nonzero().flatten()
    for t in hit_pos.tolist():
        p, r = st.pages[0][t // 64], t % 64
        assert torch.equal(eng.arena.data[p, :, :, r], want[p, :, :, r])
    eng.release(st)
