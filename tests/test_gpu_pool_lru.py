"""KV Writer parity: LRU eviction of the device pool against
an ordered-dict LRU restated from the reference's test oracle
(reference pkg/tests/oracles.py:50-74, trace test test_pool.py:136-170):
random insert / lookup-touch / evict steps, identical eviction sets and
order, identical survivors.  Also the incremental device index: after long
insert/evict churn (compaction and slot renumbering included) every lookup
equals the C oracle's pool lookup bit for bit."""
from collections import OrderedDict

import numpy as np
import pytest

from oracle import kvshare_oracle as O

pytestmark = pytest.mark.gpu


class _OrderedLRU:
    """Keys oldest-first with their byte sizes (the reference oracle's model:
    insert moves to the end, a lookup's contributors move to the end in
    their current order, eviction pops the front until the sum fits)."""

    def __init__(self):
        self.items = OrderedDict()

    def insert(self, key, size):
        self.items.pop(key, None)
        self.items[key] = size

    def touch(self, keys):
        for k in [k for k in self.items if k in keys]:
            self.items.move_to_end(k)

    def evict(self, cap):
        out = []
        while self.items and sum(self.items.values()) > cap:
            out.append(self.items.popitem(last=False)[0])
        return out


def _pool(cfg_kw=None):
    import paper_2503_16525_b200 as K
    from paper_2503_16525_b200.pool import CachePool
    cfg = K.ModelConfig(num_layers=2, num_heads=2, d_model=16, vocab_size=256, seed=0)
    return K, cfg, CachePool(cfg, K.HashParams(window_size=4), arena_pages=2048)


def test_lru_trace_equivalence():
    K, cfg, pool = _pool()
    rng = np.random.default_rng(0)
    ref = _OrderedLRU()
    token_sets = {}
    for step in range(2500):
        op = rng.choice(["insert", "touch", "evict"], p=[0.5, 0.4, 0.1])
        if op == "insert" or not token_sets:
            name = f"r{int(rng.integers(40))}"
            base = 300 + 50 * int(name[1:])
            tokens = [t % 256 for t in rng.integers(base, base + 40, 8).tolist()]
            token_sets[name] = tokens
            k = rng.normal(size=(2, 2, 8, 8))
            pool.insert(name, tokens, k, -k)
            ref.insert(name, pool.entries[name].size_bytes)
        elif op == "touch":
            name = sorted(token_sets)[int(rng.integers(len(token_sets)))]
            if name in pool.entries:
                reuse = pool.lookup(token_sets[name])
                ref.touch({e.request_id for e, _ in reuse.sources.values()})
        else:
            keep = int(rng.integers(0, len(pool.entries) + 1))
            sizes = sorted(e.size_bytes for e in pool.entries.values())
            budget = sum(sizes[:keep])
            got = pool.evict_to_capacity(budget)
            assert got == ref.evict(budget), f"step {step}"
            for name in got:
                token_sets.pop(name, None)
    assert list(pool.entries) and sorted(pool.entries) == sorted(ref.items)
    # survivors' LRU order equals the reference's
    assert [e.request_id for e in sorted(pool.entries.values(), key=lambda e: e.last_access)] \
        == list(ref.items)


def test_capacity_insert_evicts_oldest():
    """test_pool.py:125-134 pattern: a one-entry byte budget keeps the newest."""
    import paper_2503_16525_b200 as K
    from paper_2503_16525_b200.pool import CachePool
    cfg = K.ModelConfig(num_layers=2, num_heads=2, d_model=16, vocab_size=256, seed=0)
    rng = np.random.default_rng(1)
    probe = CachePool(cfg, K.HashParams(window_size=4), arena_pages=8)
    k = rng.normal(size=(2, 2, 8, 8))
    probe.insert("x", list(range(8)), k, k)
    pool = CachePool(cfg, K.HashParams(window_size=4), capacity_bytes=probe.total_bytes,
                     arena_pages=8)
    pool.insert("a", rng.integers(0, 256, 8).tolist(), k, k)
    pool.insert("b", rng.integers(0, 256, 8).tolist(), k, k)
    assert list(pool.entries) == ["b"]
    assert pool.arena.free_pages == 8 - 1          # the evicted entry's page came back


def test_incremental_index_matches_oracle_under_churn():
    K, cfg, pool = _pool()
    rng = np.random.default_rng(2)
    live = {}
    for step in range(600):
        if rng.random() < 0.6 or not live:
            name = f"e{int(rng.integers(60))}"
            n = int(rng.integers(4, 120))
            toks = rng.integers(0, 24, n).tolist()               # small alphabet: many hits
            k = np.zeros((2, 2, n, 8))
            pool.insert(name, toks, k, k)
            live[name] = toks
        else:
            names = sorted(live)
            victim = names[int(rng.integers(len(names)))]
            keep = sum(e.size_bytes for e in pool.entries.values()
                       if e.request_id != victim and e.last_access > pool.entries[victim].last_access)
            for gone in pool.evict_to_capacity(keep):
                live.pop(gone)
        if step % 25 == 0:
            req = rng.integers(0, 24, int(rng.integers(8, 200))).tolist()
            order = sorted(pool.entries.values(), key=lambda e: -e.insert_seq)
            se, sc, _ = O.pool_lookup([e.tokens for e in order], req, 4)
            reuse = pool.lookup(req)
            got = {p: (e.request_id, c) for p, (e, c) in reuse.sources.items()}
            want = {int(p): (order[se[p]].request_id, int(sc[p]))
                    for p in np.nonzero(se >= 0)[0]}
            assert got == want, f"step {step}"
    # freed slot ids were reclaimed and dead windows compacted at some point
    assert len(pool._slots) <= 2 * len(pool.entries) + 64
