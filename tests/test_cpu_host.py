"""CPU-side checks: the C ABI library loads and exports every symbol the
header declares, the host logic of the path (validation, budgets, the batch
hand-off, partitioning, the synthetic stream) and the error mapping."""
import ctypes
import math
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _lib_path():
    from paper_2503_16525_b200 import _native
    if not os.path.exists(_native.LIB_PATH):
        from paper_2503_16525_b200.build import build
        build()
    return _native.LIB_PATH


def test_library_exports_every_declared_symbol():
    with open(os.path.join(ROOT, "include", "kvshare.h")) as fh:
        header = fh.read()
    declared = set(re.findall(r"\b(kvs_[a-z0-9_]+)\s*\(", header))
    assert "kvs_pool_lookup" in declared and "kvs_attention_fwd" in declared
    lib = ctypes.CDLL(_lib_path())
    for name in sorted(declared):
        assert hasattr(lib, name), name
    lib.kvs_abi_version.restype = ctypes.c_int32
    assert lib.kvs_abi_version() == 1
    out = subprocess.run(["nm", "-D", _lib_path()], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (kvs_\w+)", out))
    assert declared <= exported


def test_native_binding_covers_header():
    from paper_2503_16525_b200 import _native
    with open(os.path.join(ROOT, "include", "kvshare.h")) as fh:
        declared = set(re.findall(r"\b(kvs_[a-z0-9_]+)\s*\(", fh.read()))
    assert declared <= set(_native.exported_symbols()) | {"kvs_embed_rows", "kvs_build_rows"}


def test_sm100a_cubin_has_tcgen05_and_tma():
    out = subprocess.run(["cuobjdump", "-sass", _lib_path()], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    sass = out.stdout
    assert "sm_100a" in sass or "SM100" in sass.upper()
    for mnemonic in ("UTCHMMA", "UTMALDG", "LDTM"):
        assert mnemonic in sass, mnemonic


def test_workspace_queries_without_gpu():
    from paper_2503_16525_b200 import _native as N
    assert N.ws_bytes("kvs_pool_lookup_workspace", 4096) >= 4096 * 16
    assert N.ws_bytes("kvs_match_pairs_workspace", 100, 50) > 0
    assert N.ws_bytes("kvs_dhd_alpha_workspace", 4096, 32, 8) >= 4096 * 40 * 4


def test_no_gpu_means_loud_failure():
    import torch
    from paper_2503_16525_b200 import DeviceError, _native
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(DeviceError):
        _native.load()


def test_hash_params_validation():
    import paper_2503_16525_b200 as K
    assert (K.HashParams().window_size, K.HashParams().base, K.HashParams().modulus) == \
        (8, 31, 1_000_000_007)
    for kw in ({"window_size": 0}, {"base": 1}, {"modulus": 30}, {"modulus": 1_000_000_008}):
        with pytest.raises(K.ParameterError):
            K.HashParams(**kw)
    K.HashParams(window_size=3, modulus=251)


def test_selection_config_and_budget():
    import paper_2503_16525_b200 as K
    from paper_2503_16525_b200.engine import budget
    assert K.SelectionConfig(ratio=0.55).budget(100) == 56
    assert K.SelectionConfig(ratio=0.3).budget(10) == 3
    assert K.SelectionConfig(ratio=0.01).budget(7) == 1
    for r in np.linspace(0.01, 1.0, 97):
        for n in (1, 7, 100, 2048, 8192):
            assert budget(float(r), n) == min(math.ceil(float(r) * n), n)
    for kw in ({"ratio": 0.0}, {"ratio": 1.5}, {"n_extra": -1}):
        with pytest.raises(K.ParameterError):
            K.SelectionConfig(**kw)


def test_schedule_matches_reference_rules():
    import paper_2503_16525_b200 as K
    from golden_io import match_doc
    for c in match_doc()["schedule"]:
        reqs = [K.Request(i, a, [], 0, h) for i, a, h in zip(c["ids"], c["arrival"], c["hit"])]
        got = K.schedule(reqs, c["batch_size"], aging_lambda=c["aging"], now_ms=c["now"])
        assert [[r.id for r in b.requests] for b in got] == c["batches"]
    with pytest.raises(K.ParameterError):
        K.schedule([], 0)
    with pytest.raises(K.ParameterError):
        K.Request("x", 0.0, [], 0, 1.5)


def test_partition_batch_balances_and_prefers_owner():
    import paper_2503_16525_b200 as K
    reqs = [K.Request(f"r{i}", float(i), [0] * 4096, 0, h)
            for i, h in enumerate([0.5, 0.5, 0.9, 0.1, 0.5, 0.5, 0.0, 0.8])]
    parts = K.partition_batch(K.Batch(reqs), 4)
    assert sorted(i for p in parts for i in p) == list(range(8))
    assert all(len(p) >= 1 for p in parts)
    owner = [[0, 0, 0, 0] for _ in reqs]
    owner[2][3] = 1000
    parts = K.partition_batch(K.Batch(reqs), 4, owner)
    assert 2 in parts[3]
    assert K.partition_batch(K.Batch(reqs), 1) == [list(range(8))]


def test_workload_hit_rate_and_determinism():
    from paper_2503_16525_b200.workload import request_batches, source_requests
    from oracle import kvshare_oracle as O
    src = source_requests(4, 2048, 128256, seed=0)
    b1 = request_batches(src, 2, 3, 2048, 0.5, 128256, seed=1)
    b2 = request_batches(src, 2, 3, 2048, 0.5, 128256, seed=1)
    assert all((x == y).all() for a, b in zip(b1, b2) for x, y in zip(a, b))
    req = b1[0][0]
    se, _, _ = O.pool_lookup(src[::-1], req, 8)
    hit = float((se >= 0).mean())
    assert 0.45 <= hit <= 0.56


def test_status_codes_map_to_reference_errors():
    from paper_2503_16525_b200 import errors as E
    assert E.STATUS_ERRORS[1] is E.ParameterError and issubclass(E.ParameterError, ValueError)
    assert E.STATUS_ERRORS[4] is E.CacheError and issubclass(E.CacheError, E.KVLabError)
    e = E.FormatError("bad", 12)
    assert e.offset == 12 and "12" in str(e)


def test_model_config_shapes():
    import paper_2503_16525_b200 as K
    cfg = K.ModelConfig(**K.LLAMA31_8B)
    assert (cfg.d_k, cfg.kv_heads, cfg.group) == (128, 8, 4)
    cfg = K.ModelConfig(**K.QWEN25_7B)
    assert (cfg.d_k, cfg.kv_heads, cfg.group) == (128, 4, 7)
    with pytest.raises(K.ConfigError):
        K.ModelConfig(num_heads=3, d_model=64)
    with pytest.raises(K.ConfigError):
        K.ModelConfig(num_heads=4, num_kv_heads=3)


def test_oracle_rope_reduces_to_reference_and_realigns():
    """RoPE restatement: rotation by 0 is identity; rotating a rotated row by
    (dst - src) equals rotating the raw row by dst (the G1 re-alignment)."""
    from oracle import kvshare_oracle as O
    tab = O.rope_table(512, 16, 10000.0)
    rng = np.random.default_rng(0)
    x = rng.normal(size=(2, 5, 16))
    np.testing.assert_allclose(O.rotate(x, np.zeros(5, int), tab), x)
    src = np.array([3, 10, 40, 7, 0])
    dst = np.array([100, 11, 2, 7, 300])
    once = O.rotate(x, dst, tab)
    twice = O.rotate(O.rotate(x, src, tab), dst - src, tab)
    np.testing.assert_allclose(once, twice, atol=1e-5)
