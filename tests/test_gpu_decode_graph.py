"""Engine.decode_graph: the decode token step (probe query, D3, chosen U
{new} rows through every layer - reference engine.py:298-328 batched)
captured once as a CUDA graph and replayed per token must equal the eager
decode_step_device bit for bit: per-step hidden rows, D3 choices, the
eligibility mask and every K/V row of the cache, on twin prefills of a
ragged batch with reuse."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _engine():
    import paper_2503_16525_b200 as K
    from paper_2503_16525_b200.engine import Engine
    from paper_2503_16525_b200.pool import CachePool
    cfg = K.ModelConfig(num_layers=3, num_heads=8, num_kv_heads=2, d_model=1024,
                        vocab_size=2048, seed=3, rope_theta=10000.0, max_positions=2048)
    model = K.init_model(cfg)
    pool = CachePool(cfg, K.HashParams(window_size=8), arena_pages=256)
    eng = Engine(model, pool)
    rng = np.random.default_rng(7)
    srcs = [rng.integers(0, 2048, 600) for _ in range(3)]
    for i, s in enumerate(srcs):
        st = eng.prefill_batch([s], mode="full")
        eng.write_back(st, [f"src{i}"])
    reqs = []
    for n in (700, 333, 1024):
        t = rng.integers(0, 2048, n)
        a = int(rng.integers(0, 300))
        t[50:50 + 250] = srcs[len(reqs)][a:a + 250]
        reqs.append(t)
    return eng, reqs


@pytest.mark.parametrize("n_extra", [3, 0])
def test_decode_graph_equals_eager(n_extra):
    eng, reqs = _engine()
    steps = 6
    toks = torch.from_numpy(np.random.default_rng(1).integers(0, 2048, (steps, len(reqs)))).cuda()
    st_e = eng.prefill_batch(reqs, ratio=0.2, decode_capacity=steps + 2)
    st_g = eng.prefill_batch(reqs, ratio=0.2, decode_capacity=steps + 2)
    assert torch.equal(st_e.eligible, st_g.eligible)
    outs_e, outs_g = [], []
    for st, outs, graph in ((st_e, outs_e, False), (st_g, outs_g, True)):
        h, ch, nc = eng.decode_step_device(st, toks[0], n_extra)        # eager first step
        outs.append((h.clone(), ch.clone(), nc.clone()))
        g = eng.decode_graph(st, n_extra) if graph else None
        for t in range(1, steps):
            h, ch, nc = g.replay(toks[t]) if graph else eng.decode_step_device(st, toks[t], n_extra)
            outs.append((h.clone(), ch.clone(), nc.clone()))
    torch.cuda.synchronize()
    for (he, ce, ne), (hg, cg, ng) in zip(outs_e, outs_g):
        assert torch.equal(ne, ng)
        assert torch.equal(ce, cg)
        assert torch.equal(he, hg)
    if n_extra:
        assert int(sum(o[2].sum() for o in outs_e)) > 0                 # D3 chose rows
    assert torch.equal(st_e.eligible, st_g.eligible)
    assert (st_e.ctx_len == st_g.ctx_len).all()
    assert torch.equal(st_e._ctx_dev, st_g._ctx_dev)
    for r in range(len(reqs)):
        n = int(st_e.ctx_len[r])
        for layer in range(3):
            for kv in (0, 1):
                assert torch.equal(eng.arena.rows(st_e.pages[r], n, layer, kv),
                                   eng.arena.rows(st_g.pages[r], n, layer, kv))
