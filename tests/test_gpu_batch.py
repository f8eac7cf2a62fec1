"""Batched device prefill (Engine.prefill_batch - the path bench.py times)
against the fp64 oracle per request: hit maps bit-exact, DHD scores within
tolerance, selections inside the tie band, and each request's last hidden
row (the first token's state) within the hidden-state tolerance of the
oracle's partial prefill with the SAME selected set.  Covers the fast path
(probe layer 0 in place, partial prefill from layer 1) and the plain path."""
import numpy as np
import pytest

from oracle import kvshare_oracle as O
from parity import HIDDEN_TOL, assert_scores_close, assert_selection_tie_band, bf16

pytestmark = pytest.mark.gpu


def _setup(L, H, kvh, d_model, rope, n_src=3, seed=0):
    import paper_2503_16525_b200 as K
    from paper_2503_16525_b200.engine import Engine
    from paper_2503_16525_b200.pool import CachePool
    cfg = K.ModelConfig(num_layers=L, num_heads=H, d_model=d_model, vocab_size=512, seed=seed,
                        num_kv_heads=kvh, rope_theta=rope, max_positions=2048)
    model = K.init_model(cfg)
    emb, layers = model.host_weights
    W = {"embedding": bf16(emb), "layers": [tuple(bf16(w) for w in l) for l in layers]}
    ocfg = O.OracleConfig(L, H, d_model, 512, seed, kvh, rope)
    table = O.rope_table(2048, cfg.d_k, rope) if rope else None
    pool = CachePool(cfg, K.HashParams(window_size=8), arena_pages=256)
    rng = np.random.default_rng(seed)
    srcs = []
    for s in range(n_src):
        src = rng.integers(0, 512, int(rng.integers(150, 400))).tolist()
        st = O.forward(src, W, ocfg, table=table)
        pool.insert(f"s{s}", src, bf16(st["k"]), bf16(st["v"]))
        srcs.append(src)
    return K, Engine(model, pool), pool, W, ocfg, table, srcs, rng


def _requests(srcs, rng, n_req):
    reqs = []
    for r in range(n_req):
        a = srcs[r % len(srcs)]
        b = srcs[(r + 1) % len(srcs)]
        t = (rng.integers(0, 512, 13).tolist() + a[20:140] + rng.integers(0, 512, 40).tolist()
             + b[5:90] + rng.integers(0, 512, 17 + r).tolist())
        reqs.append(t)
    return reqs


@pytest.mark.parametrize("L,H,kvh,d_model,rope", [(3, 8, 2, 1024, 10000.0), (2, 4, 4, 512, None),
                                                  (4, 4, 2, 512, 500000.0)])
def test_prefill_batch_vs_oracle(L, H, kvh, d_model, rope):
    K, eng, pool, W, ocfg, table, srcs, rng = _setup(L, H, kvh, d_model, rope)
    reqs = _requests(srcs, rng, 3)
    ratio = 0.3
    st = eng.prefill_batch(reqs, ratio=ratio)
    slot = st.src_slot.cpu().numpy()
    cand = st.src_cand.cpu().numpy()
    sel = st.selected.cpu().numpy().astype(bool)
    score = st.score.double().cpu().numpy()
    hidden_last = st.hidden_last.double().cpu().numpy()
    order = sorted(pool.entries.values(), key=lambda e: -e.insert_seq)
    entries = [pool.entries[e.request_id] for e in order]
    for r, t in enumerate(reqs):
        a, b = int(st.req_off_host[r]), int(st.req_off_host[r + 1])
        se, sc, _ = O.pool_lookup([e.tokens for e in order], t, 8)
        got_slot = slot[a:b]
        assert ((got_slot >= 0) == (se >= 0)).all()
        hit = se >= 0
        assert [pool.slot_entry(s).request_id for s in got_slot[hit]] == \
            [order[i].request_id for i in se[hit]]
        assert (cand[a:b][hit] == sc[hit]).all()
        oreuse = O.Reuse(se, sc, [e.k for e in entries], [e.v for e in entries])
        _, want_sel, _, info = O.prefill_with_selection(t, W, ocfg, oreuse, ratio, table)
        assert_scores_close(score[a:b][hit], info["scores"][hit])
        got = np.nonzero(sel[a:b])[0].tolist()
        assert_selection_tie_band(got, want_sel, info["scores"], O.budget(ratio, int(hit.sum())))
        # oracle partial prefill with the device's own selected set
        stt = O.forward(t, W, ocfg, oreuse, {l: set(got) for l in range(L)}, table)
        want_h = stt["hidden"][-1][-1]
        err = np.linalg.norm(hidden_last[r] - want_h) / np.linalg.norm(want_h)
        assert err < HIDDEN_TOL, f"request {r}: last hidden rel err {err:.3e}"
    eng.release(st)


def test_prefill_batch_fast_path_equals_plain_path():
    """Probe-layer-0-in-place + layer-1 start == full partial prefill (the
    reference identity: layer-0 K/V are context-free)."""
    K, eng, pool, W, ocfg, table, srcs, rng = _setup(3, 8, 2, 1024, 10000.0, seed=4)
    reqs = _requests(srcs, rng, 2)
    fast = eng.prefill_batch(reqs, ratio=0.25)
    h_fast = fast.hidden_last.double().cpu().numpy()
    sel_fast = fast.selected.cpu().numpy()
    eng.release(fast)
    eng.layer0_fast = False
    plain = eng.prefill_batch(reqs, ratio=0.25, mode="selective")
    assert (plain.selected.cpu().numpy() == sel_fast).all()
    rel = np.linalg.norm(plain.hidden_last.double().cpu().numpy() - h_fast) / np.linalg.norm(h_fast)
    assert rel < 5e-3
    eng.release(plain)
