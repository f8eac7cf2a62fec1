"""Generate pool goldens by running the REFERENCE ``kvlab`` here.

    python tests/golden/make_golden_pool.py [/root/reference/pkg/src]

(1) KVSH file:
Writes tests/golden/ref_pool.kvsh: a reference CachePool (2 layers, 2 heads,
d_k 8 - multi-head, so heads == kv_heads and the file is the reference's own
format) holding three entries inserted in order a, b, c with K/V values that
are exactly representable in bf16 (the device arena's storage type), saved
by the reference's CachePool.save (pool.py:174-189).  The device pool must
load it bit-exactly (pool.py:191-241) and save it back byte-identically.
Also writes ref_pool.json with the entries' ids, tokens and a sha256 of the
file for the test to check against.

(2) golden_fixed_chunk.json: CachePool.lookup(tokens, fixed_chunk=c)
(pool.py:125-161 -> matching.fixed_chunk_match, matching.py:171-194) on
random pools with shared blocks at aligned and unaligned offsets, duplicate
blocks and replaced ids; positions, source entry (recency rank), cand_pos and
the contributors' LRU refresh order.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = sys.argv[1] if len(sys.argv) > 1 else "/root/reference/pkg/src"
sys.path.insert(0, REF)
os.environ["KVLAB_MATCH_BACKEND"] = "pure"       # matcher backend is irrelevant to save()

from kvlab.matching import HashParams  # noqa: E402
from kvlab.model import ModelConfig  # noqa: E402
from kvlab.pool import CachePool  # noqa: E402


def bf16_exact(x: np.ndarray) -> np.ndarray:
    """Round float64 values to bf16 (RNE) and widen back (exact in f32/f64)."""
    b = x.astype(np.float32).view(np.uint32)
    b = (b + 0x7FFF + ((b >> 16) & 1)) & 0xFFFF0000
    return b.view(np.float32).astype(np.float64)


def main():
    cfg = ModelConfig(num_layers=2, num_heads=2, d_model=16, vocab_size=1000, seed=0)
    pool = CachePool(cfg)
    rng = np.random.default_rng(7)
    doc = {"entries": []}
    for ident, n in (("a", 9), ("b", 70), ("c", 33)):
        toks = rng.integers(0, 1000, n)
        k = bf16_exact(rng.normal(size=(2, 2, n, 8)))
        v = bf16_exact(rng.normal(size=(2, 2, n, 8)))
        pool.insert(ident, toks, k, v)
        doc["entries"].append({"id": ident, "tokens": toks.tolist()})
    path = os.path.join(HERE, "ref_pool.kvsh")
    pool.save(path)
    data = open(path, "rb").read()
    doc["sha256"] = hashlib.sha256(data).hexdigest()
    doc["bytes"] = len(data)
    with open(os.path.join(HERE, "ref_pool.json"), "w") as fh:
        json.dump(doc, fh)
    print(path, len(data), doc["sha256"])
    fixed_chunk_cases()


def fixed_chunk_cases():
    cfg = ModelConfig(num_layers=1, num_heads=1, d_model=2, vocab_size=64, seed=3)
    rng = np.random.default_rng(11)
    out = []
    for trial in range(40):
        c = int(rng.choice([1, 2, 3, 4, 8, 16]))
        pool = CachePool(cfg, HashParams(window_size=4))
        alpha = int(rng.choice([2, 8, 64]))
        entries = []
        for e in range(int(rng.integers(1, 6))):
            tok = rng.integers(0, alpha, int(rng.integers(1, 70))).tolist()
            if entries and rng.uniform() < 0.6:
                src = entries[int(rng.integers(len(entries)))][1]
                a = int(rng.integers(0, len(src)))
                cut = (len(tok) // 2 // c) * c if rng.uniform() < 0.5 else len(tok) // 2
                tok = tok[:cut] + src[a:] + tok[cut:]
            name = f"e{int(rng.integers(0, 4))}"
            z = np.zeros((1, 1, len(tok), 2))
            pool.insert(name, tok, z, z)
            entries.append((name, tok))
        req = rng.integers(0, alpha, int(rng.integers(0, 90))).tolist()
        if entries and rng.uniform() < 0.8:
            src = entries[int(rng.integers(len(entries)))][1]
            a, b = sorted(rng.integers(0, len(src) + 1, 2).tolist())
            if rng.uniform() < 0.5:
                a = (a // c) * c
            cut = (len(req) // 3 // c) * c
            req = req[:cut] + src[a:b] + req[cut:]
        before = {e.request_id: e.last_access for e in pool.entries.values()}
        order = [e.request_id for e in sorted(pool.entries.values(), key=lambda e: -e.insert_seq)]
        reuse = pool.lookup(req, fixed_chunk=c)
        touched = sorted([rid for rid, e in pool.entries.items() if e.last_access != before[rid]],
                         key=lambda r: pool.entries[r].last_access)
        out.append({
            "chunk": c,
            "entries_newest_first": [[int(x) for x in pool.entries[r].tokens] for r in order],
            "entry_ids_newest_first": order,
            "request": [int(x) for x in req],
            "positions": sorted(int(p) for p in reuse.sources),
            "src_entry": [order.index(reuse.sources[p][0].request_id) for p in sorted(reuse.sources)],
            "src_cand": [int(reuse.sources[p][1]) for p in sorted(reuse.sources)],
            "contributors_lru_order": touched,
        })
    with open(os.path.join(HERE, "golden_fixed_chunk.json"), "w") as fh:
        json.dump(out, fh, separators=(",", ":"))
    print("fixed-chunk cases:", len(out), "with hits:", sum(1 for o in out if o["positions"]))


if __name__ == "__main__":
    main()
