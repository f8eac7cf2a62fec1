"""Parity at the benched configurations (VERDICT r1 "Next" 1).

The path bench.py times - ``Engine.prefill_batch`` on the fast path (probe
layer 0 in place, partial prefill from layer 1, G1 on the side stream,
request-major A1 tiles, the fused D2 select) - run at the benchmark's model
widths against the float64 oracle on the same bf16 weights:

* cfg2: Llama-3.1-8B width (H=32, kv_heads=8, d=128, d_model=4096, RoPE
  theta 5e5), two 4096-token requests at 50% chunk hit from 4096-token
  sources, r = 0.2, two layers (the oracle's depth bound; every layer >= 1
  runs the same kernels).
* cfg3: Qwen2.5-7B width (H=28, kv_heads=4 -> GQA group 7, the single-head
  fwd6 attention path, d_model=3584, RoPE theta 1e6), one 8192-token request
  at 50% hit, r = 0.2, then 8 decode steps through ``Engine.decode_step``
  (probe query, D3, chosen U {new} pass) against ``oracle.Session``.

Pool entries are written by the engine itself (full-recompute prefill and
zero-copy write-back, as in bench.py); the oracle reads the same cached bf16
rows back through ``KVEntry.k/.v``.  Bars (parity.py): hit maps bit-exact,
scores <= 1.5e-2 of max, selections inside the tie band, last hidden row
(the first token's state) relative Frobenius <= 2e-2, decode hidden <= 3e-2.
"""
import numpy as np
import pytest

from oracle import kvshare_oracle as O
from parity import HIDDEN_TOL, assert_rel_fro, assert_scores_close, assert_selection_tie_band, bf16

pytestmark = pytest.mark.gpu


def _setup(shape, layers, vocab, seq, n_src, extra_tokens=0, seed=0):
    import paper_2503_16525_b200 as K
    from paper_2503_16525_b200.engine import Engine
    from paper_2503_16525_b200.pool import CachePool, KVArena
    from paper_2503_16525_b200.workload import source_requests
    cfg = K.ModelConfig(**dict(shape, num_layers=layers, vocab_size=vocab), seed=seed,
                        max_positions=seq + 64)
    model = K.init_model(cfg)                                   # reference Philox draw
    emb, lw = model.host_weights
    W = {"embedding": bf16(emb), "layers": [tuple(bf16(w) for w in l) for l in lw]}
    ocfg = O.OracleConfig(layers, cfg.num_heads, cfg.d_model, vocab, seed, cfg.kv_heads,
                          cfg.rope_theta)
    table = O.rope_table(seq + 64, cfg.d_k, cfg.rope_theta)
    pages = (n_src + 4) * ((seq + extra_tokens + 63) // 64) + 8
    pool = CachePool(cfg, K.HashParams(window_size=8), arena=KVArena(cfg, pages))
    eng = Engine(model, pool)
    sources = source_requests(n_src, seq, vocab, seed=seed)
    st = eng.prefill_batch(sources, mode="full")                # sources as bench.py builds them
    eng.write_back(st, [f"src{i}" for i in range(n_src)])
    order = sorted(pool.entries.values(), key=lambda e: -e.insert_seq)
    return K, cfg, eng, pool, W, ocfg, table, sources, order


def _oracle_reuse(order, request):
    se, sc, _ = O.pool_lookup([e.tokens for e in order], request, 8)
    return O.Reuse(se, sc, [e.k for e in order], [e.v for e in order])


def _check_hits(st, r, pool, order, oreuse):
    a, b = int(st.req_off_host[r]), int(st.req_off_host[r + 1])
    slot = st.src_slot[a:b].cpu().numpy()
    cand = st.src_cand[a:b].cpu().numpy()
    hit = oreuse.src_entry >= 0
    assert ((slot >= 0) == hit).all(), "hit map differs"
    assert [pool.slot_entry(int(s)).request_id for s in slot[hit]] == \
        [order[i].request_id for i in oreuse.src_entry[hit]], "source entries differ"
    assert (cand[hit] == oreuse.src_cand[hit]).all(), "cached positions differ"
    return a, b


def _oracle_probe_select(req, W, ocfg, oreuse, ratio, table):
    """engine.py:233-243 restated: perturbed probe at layer 1, scores, top-B."""
    reused = oreuse.reused
    q, kt, vt, kp, vp = O.perturbed_probe(req, W, ocfg, oreuse, 1, table)
    dk = O.restrict_rows(kp - kt, set(reused))
    dv = O.restrict_rows(vp - vt, set(reused))
    want_sel, scores = O.select_prefill(q, kt + dk, dv, reused, ratio, group=ocfg.group)
    return want_sel, scores, vt


def test_cfg2_llama_width_prefill_batch():
    """cfg2 (bench.py's default workload) at Llama-3.1-8B width, 2 x 4096."""
    from paper_2503_16525_b200.workload import target_request
    K, cfg, eng, pool, W, ocfg, table, sources, order = _setup(
        K_shape("llama"), layers=2, vocab=4096, seq=4096, n_src=3)
    rng = np.random.default_rng(7)
    reqs = [target_request(sources, 4096, 0.5, 4096, rng) for _ in range(2)]
    ratio = 0.2
    st = eng.prefill_batch(reqs, ratio=ratio)
    assert st.session_first == 1, "bench fast path not taken"
    sel = st.selected.cpu().numpy().astype(bool)
    score = st.score.double().cpu().numpy()
    hidden_last = st.hidden_last.double().cpu().numpy()
    budgets = st.budgets
    for r, req in enumerate(reqs):
        oreuse = _oracle_reuse(order, req)
        a, b = _check_hits(st, r, pool, order, oreuse)
        n_r = len(oreuse.reused)
        assert 0.4 * 4096 < n_r < 0.6 * 4096
        assert budgets[r] == O.budget(ratio, n_r)
        want_sel, scores, _ = _oracle_probe_select(req, W, ocfg, oreuse, ratio, table)
        hit = oreuse.src_entry >= 0
        assert_scores_close(score[a:b][hit], scores[hit])
        got = np.nonzero(sel[a:b])[0].tolist()
        assert_selection_tie_band(got, want_sel, scores, O.budget(ratio, n_r))
        fr = O.forward_rows(req, W, ocfg, oreuse, got, table=table)
        want_h = fr["hidden"][-1][-1]                            # row n-1 of the last layer
        err = np.linalg.norm(hidden_last[r] - want_h) / np.linalg.norm(want_h)
        assert err < HIDDEN_TOL, f"request {r}: last hidden rel err {err:.3e}"
        # the request's K/V cache after prefill (layer 1: reused-unselected rows
        # re-aligned cached rows, the rest fresh) equals the oracle's
        kc = eng.arena.rows(st.pages[r], 4096, 1, 0)
        vc = eng.arena.rows(st.pages[r], 4096, 1, 1)
        m = eng.model
        assert_rel_fro(m.unpad_heads(kc).double().permute(1, 0, 2).cpu().numpy(), fr["k"][1])
        assert_rel_fro(m.unpad_heads(vc).double().permute(1, 0, 2).cpu().numpy(), fr["v"][1])
    eng.release(st)


def K_shape(name):
    import paper_2503_16525_b200 as K
    return {"llama": K.LLAMA31_8B, "qwen": K.QWEN25_7B, "yi": K.YI15_9B}[name]


def test_cfg3_qwen_width_prefill_and_decode():
    """cfg3 at Qwen2.5-7B width (GQA group 7 -> fwd6), 8192 tokens, then
    8 decode-stage DHD steps against oracle.Session."""
    import torch
    from paper_2503_16525_b200.workload import target_request
    seq, n_dec, n_extra, ratio = 8192, 8, 3, 0.2
    K, cfg, eng, pool, W, ocfg, table, sources, order = _setup(
        K_shape("qwen"), layers=2, vocab=4096, seq=seq, n_src=2, extra_tokens=n_dec + 1)
    assert cfg.group == 7
    rng = np.random.default_rng(11)
    req = target_request(sources, seq, 0.5, 4096, rng)
    st = eng.prefill_batch([req], ratio=ratio, decode_capacity=n_dec + 1)
    assert st.session_first == 1
    oreuse = _oracle_reuse(order, req)
    _check_hits(st, 0, pool, order, oreuse)
    want_sel, scores, v_true = _oracle_probe_select(req, W, ocfg, oreuse, ratio, table)
    hit = oreuse.src_entry >= 0
    assert_scores_close(st.score.double().cpu().numpy()[hit], scores[hit])
    got = np.nonzero(st.selected.cpu().numpy())[0].tolist()
    assert_selection_tie_band(got, want_sel, scores, O.budget(ratio, len(oreuse.reused)))
    fr = O.forward_rows(req, W, ocfg, oreuse, got, table=table)
    want_h = fr["hidden"][-1][-1]
    h = st.hidden_last.double().cpu().numpy()[0]
    assert np.linalg.norm(h - want_h) / np.linalg.norm(want_h) < HIDDEN_TOL
    # decode stage: engine.py:298-328 vs the restated session
    osess = O.Session(req, W, ocfg, fr, oreuse.reused, got, table)
    osess._truth = v_true                                      # engine.py:81-89, from the probe
    eligible = set(oreuse.reused) - set(got)
    for step, tok in enumerate(rng.integers(0, 4096, n_dec).tolist()):
        q_t = osess.query_rows_probe(tok)
        want, dscores = O.select_decode_step(q_t, osess.k[osess.probe_layer],
                                             osess.delta_v_probe(), eligible, n_extra,
                                             group=ocfg.group)
        hd, chosen = eng.decode_step(st, [tok], n_extra)
        assert_selection_tie_band(chosen[0], want, dscores, len(want))
        osess.recompute_positions(chosen[0])
        eligible -= set(chosen[0])
        h_ref = osess.append(tok)
        assert_rel_fro(hd[0].double().cpu().numpy(), h_ref, 3e-2)
    assert int(st.eligible.sum().item()) == len(eligible)
    torch.cuda.synchronize()
    eng.release(st)
