"""R1/R2 parity on the GPU: bit-exact against the reference's golden vectors
and the C oracle (window hashes, match_pairs claim order, pool lookup)."""
import numpy as np
import pytest

from golden_io import match_doc
from oracle import kvshare_oracle as O

pytestmark = pytest.mark.gpu
DOC = match_doc()


def test_window_hashes_golden():
    from paper_2503_16525_b200 import _matchcore
    for c in DOC["hashes"]:
        got = _matchcore.window_hashes(np.array(c["tokens"], dtype=np.int64), c["w"], c["b"], c["m"])
        assert [int(x) for x in got] == c["hashes"]


def test_match_pairs_golden_all():
    from paper_2503_16525_b200 import _matchcore
    for c in DOC["match"]:
        tm, cm = _matchcore.match_pairs(np.array(c["target"], dtype=np.int64),
                                        np.array(c["candidate"], dtype=np.int64),
                                        c["w"], c["b"], c["m"])
        assert (tm, cm) == (c["tm"], c["cm"]), (c["w"], c["m"], len(c["target"]))


def test_match_sequences_api_and_known_answers():
    import paper_2503_16525_b200 as K
    p3 = K.HashParams(window_size=3)
    r = K.match_sequences([5, 6, 7, 8, 9], [1, 2, 6, 7, 8, 3], p3)   # test_matching.py:86-89
    assert r.target_matches == [1, 2, 3] and r.candidate_matches == [2, 3, 4]
    assert K.rolling_hash([1, 2, 3], 0, p3) == 1026
    assert len(K.match_sequences([1, 2], [1, 2], p3)) == 0
    assert K.build_hash_index([7, 7, 7, 7], K.HashParams(window_size=2)) == {
        int(K.window_hashes([7, 7], K.HashParams(window_size=2))[0]): [0, 1, 2]}


@pytest.mark.parametrize("seed", range(6))
def test_match_pairs_random_vs_oracle(seed):
    from paper_2503_16525_b200 import _matchcore
    rng = np.random.default_rng(seed)
    for _ in range(40):
        w = int(rng.integers(1, 9))
        m = int(rng.choice([1_000_000_007, 251, 37, 2_305_843_009_213_693_951]))
        alpha = int(rng.choice([2, 8, 1000, 2**40]))
        t = rng.integers(0, alpha, int(rng.integers(0, 300)))
        c = rng.integers(0, alpha, int(rng.integers(0, 300)))
        if t.size > 20 and c.size > 20 and rng.uniform() < 0.6:
            a = int(rng.integers(0, t.size - 10))
            c[5:5 + min(40, t.size - a)] = t[a:a + min(40, t.size - a)][:c[5:5 + 40].size]
        got = _matchcore.match_pairs(t, c, w, 31, m)
        want = O.match_pairs(t, c, w, 31, m)
        assert got == want


def test_match_pairs_large_shared_spans():
    from paper_2503_16525_b200 import _matchcore
    rng = np.random.default_rng(7)
    n = 16384
    t = rng.integers(0, 128256, n)
    c = rng.integers(0, 128256, n)
    c[1000:9000] = t[3000:11000]
    c[12000:12500] = t[100:600]
    got = _matchcore.match_pairs(t, c, 8, 31, 1_000_000_007)
    assert got == O.match_pairs(t, c, 8, 31, 1_000_000_007)
    assert len(got[0]) >= 8500


def _pool(cfg_kw=None, w=4, m=1_000_000_007):
    import paper_2503_16525_b200 as K
    from paper_2503_16525_b200.pool import CachePool
    cfg = K.ModelConfig(num_layers=1, num_heads=1, d_model=2, vocab_size=4096, seed=3)
    return cfg, CachePool(cfg, K.HashParams(window_size=w, modulus=m), arena_pages=512)


@pytest.mark.parametrize("idx", range(len(DOC["lookup"])))
def test_pool_lookup_golden(idx):
    c = DOC["lookup"][idx]
    cfg, pool = _pool(w=c["w"], m=c["m"])
    ids = c["entry_ids_newest_first"]
    for rid, tok in reversed(list(zip(ids, c["entries_newest_first"]))):
        z = np.zeros((1, 1, len(tok), 2))
        pool.insert(rid, tok, z, z)
    reuse = pool.lookup(c["request"])
    assert sorted(reuse.sources) == c["positions"]
    assert [ids.index(reuse.sources[p][0].request_id) for p in sorted(reuse.sources)] == c["src_entry"]
    assert [reuse.sources[p][1] for p in sorted(reuse.sources)] == c["src_cand"]
    assert reuse.hit_rate == pytest.approx(c["hit_rate"], abs=0)
    reuse.validate(c["request"])


def test_pool_lookup_batched_equals_single():
    cfg, pool = _pool(w=8)
    rng = np.random.default_rng(3)
    entries = []
    for e in range(12):
        tok = rng.integers(0, 4096, int(rng.integers(50, 700)))
        if entries and e % 2:
            src = entries[int(rng.integers(len(entries)))]
            tok[10:10 + min(200, src.size)] = src[:200][:tok[10:210].size]
        z = np.zeros((1, 1, tok.size, 2))
        pool.insert(f"e{e}", tok, z, z)
        entries.append(tok)
    reqs = []
    for r in range(9):
        q = rng.integers(0, 4096, int(rng.integers(20, 900)))
        src = entries[int(rng.integers(len(entries)))]
        k = min(300, q.size - 5, src.size)
        q[5:5 + k] = src[:k]
        reqs.append(q)
    import torch
    flat = torch.from_numpy(np.concatenate(reqs)).cuda()
    off = np.zeros(len(reqs) + 1, dtype=np.int64)
    off[1:] = np.cumsum([q.size for q in reqs])
    res = pool.lookup_device(flat, torch.from_numpy(off).cuda(), off)
    slot = res.src_slot.cpu().numpy()
    cand = res.src_cand.cpu().numpy()
    order = sorted(pool.entries.values(), key=lambda e: -e.insert_seq)
    for r, q in enumerate(reqs):
        se, sc, _ = O.pool_lookup([e.tokens for e in order], q, 8)
        got_slot = slot[off[r]:off[r + 1]]
        want_slot = np.array([order[e].slot if e >= 0 else -1 for e in se])
        np.testing.assert_array_equal(got_slot, want_slot)
        np.testing.assert_array_equal(cand[off[r]:off[r + 1]], sc)
    assert res.n_hit.cpu().numpy().tolist() == [int((slot[off[r]:off[r + 1]] >= 0).sum())
                                                for r in range(len(reqs))]


def test_most_recent_entry_wins_and_lru():
    cfg, pool = _pool(w=4)
    span = list(range(100, 108))
    z = np.zeros((1, 1, 8, 2))
    pool.insert("old", span, z, z)
    pool.insert("new", span, z, z)
    reuse = pool.lookup(span)
    assert {e.request_id for e, _ in reuse.sources.values()} == {"new"}
    assert pool.entries["new"].last_access > pool.entries["old"].last_access


def _fixed_doc():
    import json
    import os
    return json.load(open(os.path.join(os.path.dirname(__file__), "golden",
                                       "golden_fixed_chunk.json")))


@pytest.mark.parametrize("idx", range(40))
def test_fixed_chunk_lookup_golden(idx):
    """F5 kvs_fixed_chunk_lookup against the reference's fixed-chunk pool
    lookups (pool.py:139-159, matching.py:171-194), bit-exact, including
    which entries get their LRU tick refreshed and in what order."""
    c = _fixed_doc()[idx]
    cfg, pool = _pool(w=4)
    ids = c["entry_ids_newest_first"]
    for rid, tok in reversed(list(zip(ids, c["entries_newest_first"]))):
        z = np.zeros((1, 1, len(tok), 2))
        pool.insert(rid, tok, z, z)
    before = {rid: e.last_access for rid, e in pool.entries.items()}
    reuse = pool.lookup(c["request"], fixed_chunk=c["chunk"])
    assert sorted(reuse.sources) == c["positions"]
    assert [ids.index(reuse.sources[p][0].request_id) for p in sorted(reuse.sources)] == c["src_entry"]
    assert [reuse.sources[p][1] for p in sorted(reuse.sources)] == c["src_cand"]
    touched = sorted([r for r, e in pool.entries.items() if e.last_access != before[r]],
                     key=lambda r: pool.entries[r].last_access)
    assert touched == c["contributors_lru_order"]


def test_fixed_chunk_lookup_vs_oracle_large():
    """Long requests and entries with many aligned repeats: kernel == oracle."""
    cfg, pool = _pool(w=8)
    rng = np.random.default_rng(9)
    entries = []
    for e in range(6):
        tok = rng.integers(0, 8, int(rng.integers(500, 3000)))
        entries.append(tok)
        z = np.zeros((1, 1, tok.size, 2))
        pool.insert(f"e{e}", tok, z, z)
    for c in (1, 4, 16, 64):
        src = entries[2]
        req = np.concatenate([rng.integers(0, 8, 3 * c), src[c * 5: c * 5 + 40 * c],
                              rng.integers(0, 8, 77)])
        order = sorted(pool.entries.values(), key=lambda e: -e.insert_seq)
        se, sc, _ = O.fixed_chunk_lookup([e.tokens for e in order], req, c)
        reuse = pool.lookup(req, fixed_chunk=c)
        pos = np.nonzero(se >= 0)[0].tolist()
        assert sorted(reuse.sources) == pos
        assert [reuse.sources[p][1] for p in pos] == sc[pos].tolist()
        assert [order.index(reuse.sources[p][0]) for p in pos] == se[pos].tolist()
