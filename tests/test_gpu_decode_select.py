"""D3 (kvs_dhd_decode_select, the fused decode-stage DHD kernel) on ragged
decode batches against the oracle's select_decode_step (reference
selection.py:80-105) per request: unmasked softmax over each request's whole
context at the probe layer, mean over query heads (GQA), times the prefill
rows' dv-L1, top min(n_extra, #eligible) eligible rows ascending, chosen rows
cleared from the eligibility mask.  Cases: Llama (32/8) and Qwen (28/4)
head shapes, contexts from 1 to 9000 tokens with decode rows past the
prefill, empty / tiny eligible sets, n_extra 1..16, repeated calls on one
workspace (self-resetting counters)."""
import numpy as np
import pytest

from oracle import kvshare_oracle as O
from parity import assert_scores_close, assert_selection_tie_band

pytestmark = pytest.mark.gpu


def _batch(H, G, ctx, n_pre, seed=0):
    import torch

    from paper_2503_16525_b200 import _native as N
    from paper_2503_16525_b200.engine import Engine
    import paper_2503_16525_b200 as K
    from paper_2503_16525_b200.pool import CachePool, KVArena
    cfg = K.ModelConfig(num_layers=2, num_heads=H, num_kv_heads=G, d_model=H * 128,
                        vocab_size=64, max_positions=max(ctx) + 64)
    pages = sum((c + 63) // 64 for c in ctx) + 4
    arena = KVArena(cfg, pages)
    eng = Engine(K.ToyModel(cfg, init="device"), CachePool(cfg, arena=arena))
    st = eng.new_batch([np.zeros(n, dtype=np.int64) for n in n_pre],
                       decode_capacity=max(c - n for c, n in zip(ctx, n_pre)))
    g = torch.Generator(device="cuda").manual_seed(seed)
    arena.data.copy_((torch.randn(arena.data.shape, generator=g, device="cuda") * 0.5)
                     .to(torch.bfloat16))
    st.ctx_len = np.asarray(ctx, dtype=np.int64)
    n_tot = int(sum(n_pre))
    rng = np.random.default_rng(seed)
    st.dv_l1 = torch.from_numpy(rng.uniform(0.0, 2.0, n_tot).astype(np.float32)).cuda()
    return K, N, eng, st, rng


@pytest.mark.parametrize("H,G,ctx,n_pre,n_extra", [
    (32, 8, [4096, 4100, 1, 63, 64, 65, 700, 9000], [4090, 4096, 1, 63, 50, 65, 700, 8990], 3),
    (28, 4, [2048, 129, 3000], [2040, 100, 3000], 5),
    (32, 8, [300] * 40, [290] * 40, 16),
    (32, 8, [1000, 1000], [1000, 1000], 1),
])
def test_decode_select_batched_vs_oracle(H, G, ctx, n_pre, n_extra):
    import torch
    K, N, eng, st, rng = _batch(H, G, ctx, n_pre)
    R = len(ctx)
    q = (torch.randn(R, H, 128, device="cuda") * 0.3).to(torch.bfloat16)
    elig = np.zeros(int(sum(n_pre)), dtype=np.uint8)
    want_elig = []
    for r in range(R):
        a = int(st.req_off_host[r])
        n = n_pre[r]
        kind = r % 4
        m = rng.random(n) < (0.4 if kind < 2 else (0.0 if kind == 2 else 0.002))
        elig[a:a + n] = m
        want_elig.append(set(np.nonzero(m)[0].tolist()))
    st.eligible = torch.from_numpy(elig).cuda()
    dvl = st.dv_l1.cpu().numpy().astype(np.float64)
    for call in range(2):                                  # second call: counters reset
        chosen = eng.decode_select(st, q, n_extra)
        qh = q.double().cpu().numpy()
        for r in range(R):
            a = int(st.req_off_host[r])
            k = eng.arena.rows(st.pages[r], ctx[r], 1, 0).double().permute(1, 0, 2).cpu().numpy()
            dv = np.zeros((G, ctx[r], 128))
            dv[0, :n_pre[r], 0] = dvl[a:a + n_pre[r]]             # L1 sum == dv-L1 row
            want, scores = O.select_decode_step(qh[r], k, dv, want_elig[r], n_extra,
                                                group=H // G)
            assert_selection_tie_band(chosen[r], want, scores, len(want))
            want_elig[r] -= set(chosen[r])
        got_elig = st.eligible.cpu().numpy()
        for r in range(R):
            a = int(st.req_off_host[r])
            assert set(np.nonzero(got_elig[a:a + n_pre[r]])[0].tolist()) == want_elig[r]
    eng.release(st)


def test_decode_select_scores_output():
    """The nullable scores output holds every context row's score (decode
    rows 0), equal to the oracle's scores."""
    import paper_2503_16525_b200 as K
    rng = np.random.default_rng(3)
    for H, G, n in ((32, 8, 5000), (28, 4, 777), (4, 4, 64)):
        q_t = rng.normal(size=(H, 128)) * 0.3
        k = rng.normal(size=(G, n, 128))
        dv = rng.normal(size=(G, n, 128)) * 0.1
        elig = set(rng.choice(n, size=n // 4, replace=False).tolist())
        res = K.select_decode_step(q_t, k, dv, elig, 7)
        want, scores = O.select_decode_step(q_t, k, dv, elig, 7, group=H // G)
        assert_scores_close(res.scores, scores)
        assert_selection_tie_band(res.indices, want, scores, 7)


def test_shared_workspace_across_paths():
    """The fused kernel and the two-kernel fallback (odd head counts) share one
    workspace: the fallback's buffers sit after the fused kernel's counter
    header, so a fused call after a fallback call still starts from zeroed
    counters (regression: the fallback wrote logits over the work ticket)."""
    import paper_2503_16525_b200 as K
    rng = np.random.default_rng(11)
    for H, G, n, n_extra in ((32, 8, 3000, 7), (1, 1, 300, 3), (2, 2, 50, 3),
                             (3, 1, 900, 5), (4, 4, 64, 2), (28, 4, 777, 3)):
        q_t = rng.normal(size=(H, 128)) * 0.3
        k = rng.normal(size=(G, n, 128))
        dv = rng.normal(size=(G, n, 128)) * 0.1
        elig = set(rng.choice(n, size=n // 3, replace=False).tolist())
        res = K.select_decode_step(q_t, k, dv, elig, n_extra)
        want, scores = O.select_decode_step(q_t, k, dv, elig, n_extra, group=H // G)
        assert_scores_close(res.scores, scores)
        assert_selection_tie_band(res.indices, want, scores, n_extra)


def test_engine_workspace_across_batch_sizes():
    """One engine, one D3 workspace, batches of 100 / 2 / 100 requests: the
    small batch's logits must not land on the large batch's per-request
    counters (the counter header has one fixed size)."""
    import torch

    import paper_2503_16525_b200 as K
    from paper_2503_16525_b200.engine import Engine
    from paper_2503_16525_b200.pool import CachePool, KVArena
    H, G, n_extra = 32, 8, 3
    cfg = K.ModelConfig(num_layers=2, num_heads=H, num_kv_heads=G, d_model=H * 128,
                        vocab_size=64, max_positions=512)
    arena = KVArena(cfg, 2 * 102 * 3 + 8)
    eng = Engine(K.ToyModel(cfg, init="device"), CachePool(cfg, arena=arena))
    g = torch.Generator(device="cuda").manual_seed(5)
    arena.data.copy_((torch.randn(arena.data.shape, generator=g, device="cuda") * 0.5)
                     .to(torch.bfloat16))
    rng = np.random.default_rng(5)

    def run(R, ctx):
        st = eng.new_batch([np.zeros(ctx, dtype=np.int64)] * R, decode_capacity=0)
        st.ctx_len = np.full(R, ctx, dtype=np.int64)
        n_tot = R * ctx
        st.dv_l1 = torch.from_numpy(rng.uniform(0.0, 2.0, n_tot).astype(np.float32)).cuda()
        elig = (rng.random(n_tot) < 0.3).astype(np.uint8)
        st.eligible = torch.from_numpy(elig).cuda()
        q = (torch.randn(R, H, 128, device="cuda") * 0.3).to(torch.bfloat16)
        chosen = eng.decode_select(st, q, n_extra)
        qh, dvl = q.double().cpu().numpy(), st.dv_l1.cpu().numpy().astype(np.float64)
        for r in range(R):
            a = int(st.req_off_host[r])
            k = eng.arena.rows(st.pages[r], ctx, 1, 0).double().permute(1, 0, 2).cpu().numpy()
            dv = np.zeros((G, ctx, 128))
            dv[0, :, 0] = dvl[a:a + ctx]
            want, scores = O.select_decode_step(qh[r], k, dv,
                                                set(np.nonzero(elig[a:a + ctx])[0].tolist()),
                                                n_extra, group=H // G)
            assert_selection_tie_band(chosen[r], want, scores, len(want))
        eng.release(st)

    run(100, 130)
    run(2, 300)
    run(100, 130)
