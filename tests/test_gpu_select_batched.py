"""D2 (kvs_dhd_select, one fused launch per scheduled batch) on batches that
exercise its work distribution and all three top-B paths: many requests of
ragged lengths (1 token up to past the shared-memory key limit of 47104),
requests with no reused rows, with every row reused, budgets of 0 and of
the whole reused set, and alpha drawn from a few values so scores tie
exactly.  dv-L1 is checked against torch, scores against alpha x dv-L1 and
the selected set against the (-score, position) order of selection.py:63-66
applied to the device's own scores (bit-exact)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _case(lengths, seed):
    import paper_2503_16525_b200 as K
    from paper_2503_16525_b200.engine import Engine
    from paper_2503_16525_b200.pool import CachePool, KVArena
    dev = torch.device("cuda", 0)
    shape = dict(K.LLAMA31_8B)
    shape.update(num_layers=2, vocab_size=1000)
    cfg = K.ModelConfig(**shape, max_positions=max(lengths) + 64)
    pages = sum((n + 63) // 64 for n in lengths)
    arena = KVArena(cfg, pages + 8)
    eng = Engine(K.ToyModel(cfg, init="device"), CachePool(cfg, arena=arena))
    rng = np.random.default_rng(seed)
    st = eng.new_batch([rng.integers(0, 1000, n) for n in lengths])
    gen = torch.Generator(device=dev).manual_seed(seed)
    arena.data.normal_(generator=gen)
    n = sum(lengths)
    src = np.full(n, -1, dtype=np.int32)
    off = np.concatenate([[0], np.cumsum(lengths)])
    for r, ln in enumerate(lengths):
        mode = r % 4
        if mode == 0:
            continue                                   # nothing reused
        if mode == 1:
            src[off[r]:off[r + 1]] = 0                 # everything reused
            continue
        p = 0
        while p < ln:                                  # spans, ~half reused
            span = int(rng.integers(1, 300))
            if rng.random() < 0.5:
                src[off[r] + p: off[r] + min(ln, p + span)] = 0
            p += span
    st.src_slot = torch.from_numpy(src).to(dev)
    v_true = (torch.randn(n, cfg.kv_heads, 128, device=dev, generator=gen) * 0.5).to(torch.bfloat16)
    alpha = torch.from_numpy(rng.choice([0.0, 0.25, 0.5, 1.0], size=n).astype(np.float32)).to(dev)
    n_hit = [(src[off[r]:off[r + 1]] >= 0).sum() for r in range(len(lengths))]
    bud = []
    for r, h in enumerate(n_hit):
        choice = r % 3
        bud.append(0 if choice == 0 else int(h) if choice == 1 else
                   K.SelectionConfig(ratio=0.2).budget(int(h)) if h else 0)
    return eng, st, cfg, src, off, v_true, alpha, np.asarray(bud, np.int32)


@pytest.mark.parametrize("lengths,seed", [
    ([1, 17, 64, 65, 300, 1000, 4096, 4097], 0),
    ([4096] * 40, 1),
    ([9000, 47104, 47105, 50000], 2),
    (list(np.random.default_rng(7).integers(1, 6000, 150)), 3),
])
def test_select_batched_vs_reference(lengths, seed):
    eng, st, cfg, src, off, v_true, alpha, bud = _case([int(x) for x in lengths], seed)
    dv, score, sel = eng._select(st, v_true, alpha, bud)
    torch.cuda.synchronize()
    n = int(off[-1])
    layer = eng.probe_layer
    bt = st.block_table.cpu().numpy()
    req = np.repeat(np.arange(len(off) - 1), np.diff(off))
    pos = np.arange(n) - off[req]
    pg = torch.from_numpy(bt[req, pos // 64].astype(np.int64)).to(v_true.device)
    vc = eng.arena.data[:, layer, 1][pg, torch.from_numpy(pos % 64).to(v_true.device)]
    want_dv = (vc.float() - v_true.float()).abs().sum(dim=(1, 2))
    live = torch.from_numpy(src >= 0).to(v_true.device)
    want_dv[~live] = 0
    assert torch.allclose(dv, want_dv, rtol=1e-5, atol=1e-3)
    assert torch.equal(score, alpha * dv)
    s_dev = score.cpu().numpy()
    got = sel.cpu().numpy().astype(bool)
    for r in range(len(off) - 1):
        sl = slice(off[r], off[r + 1])
        reused = np.nonzero(src[sl] >= 0)[0]
        order = sorted(reused, key=lambda i: (-s_dev[sl][i], i))[:bud[r]]
        want = np.zeros(off[r + 1] - off[r], bool)
        want[order] = True
        assert (want == got[sl]).all(), f"request {r} (len {off[r + 1] - off[r]}, B={bud[r]})"


def test_select_batched_repeat_launches():
    """The fused launch keeps self-resetting counters in its workspace: many
    back-to-back launches on one workspace give identical results."""
    eng, st, cfg, src, off, v_true, alpha, bud = _case([3000, 4096, 700, 5000, 64], 5)
    first = [t.clone() for t in eng._select(st, v_true, alpha, bud)]
    for _ in range(20):
        out = eng._select(st, v_true, alpha, bud)
    torch.cuda.synchronize()
    for a, b in zip(first, out):
        assert torch.equal(a, b)
