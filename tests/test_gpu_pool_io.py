"""F3: KVSH pool files (reference pool.py:8-17, 174-241) through the device
arena - the reference's own file loads bit-exactly and saves back
byte-identically; round trips, GQA pools and every FormatError / CacheError
path of the reference loader."""
import hashlib
import json
import os
import struct

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _pool(L=2, H=2, d_model=16, kvh=None, pages=64):
    import paper_2503_16525_b200 as K
    from paper_2503_16525_b200.pool import CachePool
    cfg = K.ModelConfig(num_layers=L, num_heads=H, d_model=d_model, vocab_size=1000,
                        num_kv_heads=kvh)
    return CachePool(cfg, arena_pages=pages)


def _bf16(x):
    b = np.asarray(x, np.float32).view(np.uint32)
    b = (b + 0x7FFF + ((b >> 16) & 1)) & 0xFFFF0000
    return b.view(np.float32).astype(np.float64)


def test_reference_file_loads_and_saves_byte_identically(tmp_path):
    doc = json.load(open(os.path.join(GOLD, "ref_pool.json")))
    pool = _pool().load(os.path.join(GOLD, "ref_pool.kvsh"))
    assert list(pool.entries) == [e["id"] for e in doc["entries"]]
    for e in doc["entries"]:
        assert pool.entries[e["id"]].tokens.tolist() == e["tokens"]
    out = tmp_path / "again.kvsh"
    pool.save(out)
    data = out.read_bytes()
    assert len(data) == doc["bytes"]
    assert hashlib.sha256(data).hexdigest() == doc["sha256"]


def test_loaded_entries_serve_lookups():
    doc = json.load(open(os.path.join(GOLD, "ref_pool.json")))
    pool = _pool().load(os.path.join(GOLD, "ref_pool.kvsh"))
    b = doc["entries"][1]["tokens"]
    reuse = pool.lookup([5, 6, 7] + b[10:50] + [1, 2])
    assert sorted(reuse.sources) == list(range(3, 43))
    assert all(reuse.sources[p][0].request_id == "b" and reuse.sources[p][1] == p + 7
               for p in reuse.sources)


@pytest.mark.parametrize("kvh,H,d_model", [(None, 2, 16), (2, 8, 256), (1, 4, 512)])
def test_round_trip(tmp_path, kvh, H, d_model):
    pool = _pool(L=3, H=H, d_model=d_model, kvh=kvh, pages=128)
    cfg = pool.config
    rng = np.random.default_rng(H)
    want = {}
    for ident, n in (("x", 1), ("y", 64), ("z", 200)):
        toks = rng.integers(0, 1000, n)
        k = _bf16(rng.normal(size=(3, cfg.kv_heads, n, cfg.d_k)))
        v = _bf16(rng.normal(size=(3, cfg.kv_heads, n, cfg.d_k)))
        pool.insert(ident, toks, k, v)
        want[ident] = (toks, k, v)
    path = tmp_path / "p.kvsh"
    pool.save(path)
    again = _pool(L=3, H=H, d_model=d_model, kvh=kvh, pages=128).load(path)
    for ident, (toks, k, v) in want.items():
        e = again.entries[ident]
        assert e.tokens.tolist() == toks.tolist()
        np.testing.assert_array_equal(e.k, k)
        np.testing.assert_array_equal(e.v, v)
    path2 = tmp_path / "q.kvsh"
    again.save(path2)
    assert path.read_bytes() == path2.read_bytes()


def test_load_errors_match_reference(tmp_path):
    from paper_2503_16525_b200.errors import CacheError, FormatError
    data = open(os.path.join(GOLD, "ref_pool.kvsh"), "rb").read()
    pool = _pool()

    def load(blob):
        p = tmp_path / "bad.kvsh"
        p.write_bytes(blob)
        return pool.load(p)

    with pytest.raises(FormatError) as e:
        load(b"KVSX" + data[4:])
    assert e.value.offset == 0
    with pytest.raises(FormatError) as e:
        load(data[:4] + struct.pack("<I", 2) + data[8:])
    assert e.value.offset == 4
    with pytest.raises(FormatError) as e:
        load(data[:-3])
    assert "truncated" in str(e.value)
    with pytest.raises(FormatError) as e:
        load(data + b"\0")
    assert e.value.offset == len(data)
    with pytest.raises(CacheError):
        _pool(L=3).load(os.path.join(GOLD, "ref_pool.kvsh"))
    # a failed load leaves the pool as it was
    ok = _pool().load(os.path.join(GOLD, "ref_pool.kvsh"))
    with pytest.raises(FormatError):
        p = tmp_path / "t.kvsh"
        p.write_bytes(data[:100])
        ok.load(p)
    assert list(ok.entries) == ["a", "b", "c"]
