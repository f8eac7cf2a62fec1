"""Generate golden vectors by running the REFERENCE ``kvlab`` in this container.

Usage (container only - /root/reference does not exist on the GPU box):

    python tests/golden/make_golden.py [/root/reference/pkg/src]

The reference is imported from a scratch copy of its source tree with its
_matchcore.pyx cythonized there (the compiled backend the reference ships;
the pure one overflows int64 for ids >= 2**31).  Outputs, committed here:

* golden_match.json   - window hashes, match_pairs and CachePool.lookup cases
                        (reference tests' shapes: random, adversarial, forced
                        collisions at m=251, hand-traced)
* golden_model_*.npz  - Philox weights, probe tensors, DHD scores, selected
                        sets, prefill states and decode-stage choices for small
                        configs (engine.prefill_with_selection / run_generation)
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = sys.argv[1] if len(sys.argv) > 1 else "/root/reference/pkg/src"


def _compiled_reference(src: str) -> str:
    """Copy the reference package to a scratch dir and cythonize its
    _matchcore.pyx there (the pure backend overflows int64 for token ids
    >= 2**31, so goldens come from the compiled backend the reference ships)."""
    import shutil
    import subprocess
    import tempfile
    dst = os.path.join(tempfile.mkdtemp(prefix="kvlab_ref_"), "src")
    shutil.copytree(src, dst)
    inc = np.get_include()
    subprocess.check_call([sys.executable, "-m", "cython", "-3",
                           os.path.join(dst, "kvlab", "_matchcore.pyx")])
    import sysconfig
    ext = sysconfig.get_config_var("EXT_SUFFIX")
    subprocess.check_call(["gcc", "-O2", "-shared", "-fPIC",
                           "-I" + sysconfig.get_paths()["include"], "-I" + inc,
                           os.path.join(dst, "kvlab", "_matchcore.c"),
                           "-o", os.path.join(dst, "kvlab", "_matchcore" + ext)])
    return dst


sys.path.insert(0, _compiled_reference(REF))

import kvlab.matching  # noqa: E402
assert kvlab.matching.BACKEND == "compiled", kvlab.matching.BACKEND
from kvlab import engine, model as kmodel, selection  # noqa: E402
from kvlab.matching import HashParams, match_sequences, window_hashes  # noqa: E402
from kvlab.model import ModelConfig, init_model, model_forward  # noqa: E402
from kvlab.pool import CachePool  # noqa: E402
from kvlab.scheduling import Request, schedule  # noqa: E402
from kvlab.selection import SelectionConfig  # noqa: E402


def match_cases(rng):
    cases = []

    def add(t, c, w, b=31, m=1_000_000_007):
        p = HashParams(window_size=w, base=b, modulus=m)
        r = match_sequences(t, c, p)
        cases.append({"target": [int(x) for x in t], "candidate": [int(x) for x in c],
                      "w": w, "b": b, "m": m,
                      "tm": r.target_matches, "cm": r.candidate_matches})

    add([5, 6, 7, 8, 9], [1, 2, 6, 7, 8, 3], 3)                      # test_matching.py:86-89
    tok = rng.integers(0, 16, 40).tolist()
    add(tok, tok, 3)                                                  # :81-84
    for _ in range(120):                                              # :105-112
        add(rng.integers(0, 16, int(rng.integers(1, 100))).tolist(),
            rng.integers(0, 16, int(rng.integers(1, 100))).tolist(), 4)
    for t, c in [([3] * 64, [3] * 64), ([3] * 64, [3] * 5),           # :114-125
                 ([1, 2] * 32, [2, 1] * 32), ([0, 0, 0, 1] * 16, [0] * 64),
                 ([7] * 200, [7] * 150)]:
        add(t, c, 4)
    for _ in range(60):                                               # :127-138
        add(rng.integers(0, 1000, 64).tolist(), rng.integers(0, 1000, 64).tolist(), 3, 31, 251)
    for _ in range(30):
        add(rng.integers(0, 10, int(rng.integers(1, 48))).tolist(),
            rng.integers(0, 10, int(rng.integers(1, 48))).tolist(), int(rng.integers(1, 6)))
    for _ in range(20):                                               # tiny modulus 37
        add(rng.integers(0, 50, 80).tolist(), rng.integers(0, 50, 80).tolist(),
            int(rng.integers(1, 5)), 31, 37)
    # larger shared-span cases (bench_matching.py shapes)
    for n in (512, 2048):
        base = rng.integers(0, 4096, n)
        cand = rng.integers(0, 4096, n)
        cand[n // 4: n // 4 + n // 2] = base[n // 8: n // 8 + n // 2]
        add(base.tolist(), cand.tolist(), 8)
    # tokens beyond the modulus and large ids
    add((rng.integers(0, 2**40, 50)).tolist(), (rng.integers(0, 2**40, 50)).tolist(), 2)
    big = rng.integers(0, 2**33, 30).tolist()
    add(big + big, big[5:] + big, 4)
    return cases


def hash_cases(rng):
    out = []
    for n, w, m in [(3, 3, 1_000_000_007), (10, 5, 1_000_000_007), (1100, 8, 1_000_000_007),
                    (64, 8, 1_000_000_007), (200, 3, 251), (7, 8, 1_000_000_007),
                    (300, 1, 37), (500, 16, 2_147_483_647)]:
        t = rng.integers(0, 2**34 if m > 1000 else 4096, n).tolist()
        p = HashParams(window_size=w, modulus=m)
        out.append({"tokens": t, "w": w, "b": 31, "m": m,
                    "hashes": [int(h) for h in window_hashes(t, p)]})
    out.append({"tokens": [0] * 10, "w": 5, "b": 31, "m": 1_000_000_007,
                "hashes": [0] * 6})
    return out


def lookup_cases(rng):
    cfg = ModelConfig(num_layers=1, num_heads=1, d_model=2, vocab_size=4096, seed=3)
    out = []
    for trial in range(60):
        w = int(rng.integers(2, 6))
        m = 251 if trial % 5 == 0 else 1_000_000_007
        pool = CachePool(cfg, HashParams(window_size=w, modulus=m))
        alpha = int(rng.choice([4, 16, 4096]))
        entries = []
        for e in range(int(rng.integers(1, 7))):
            tok = rng.integers(0, alpha, int(rng.integers(1, 60))).tolist()
            if entries and rng.uniform() < 0.5:
                src = entries[int(rng.integers(len(entries)))][1]
                a = int(rng.integers(0, len(src)))
                tok = tok[: len(tok) // 2] + src[a:] + tok[len(tok) // 2:]
            name = f"e{int(rng.integers(0, 5))}"  # duplicate ids replace (pool.py:115)
            z = np.zeros((1, 1, len(tok), 2))
            pool.insert(name, tok, z, z)
            entries.append((name, tok))
        req = rng.integers(0, alpha, int(rng.integers(0, 80))).tolist()
        if entries and rng.uniform() < 0.7:
            src = entries[int(rng.integers(len(entries)))][1]
            a, b = sorted(rng.integers(0, len(src) + 1, 2).tolist())
            req = req[: len(req) // 3] + src[a:b] + req[len(req) // 3:]
        before = {e.request_id: e.last_access for e in pool.entries.values()}
        order = [e.request_id for e in sorted(pool.entries.values(), key=lambda e: -e.insert_seq)]
        reuse = pool.lookup(req)
        touched = sorted([rid for rid, e in pool.entries.items() if e.last_access != before[rid]],
                         key=lambda r: pool.entries[r].last_access)
        out.append({
            "w": w, "b": 31, "m": m,
            "entries_newest_first": [[int(x) for x in pool.entries[r].tokens] for r in order],
            "entry_ids_newest_first": order,
            "request": [int(x) for x in req],
            "positions": sorted(int(p) for p in reuse.sources),
            "src_entry": [order.index(reuse.sources[p][0].request_id) for p in sorted(reuse.sources)],
            "src_cand": [int(reuse.sources[p][1]) for p in sorted(reuse.sources)],
            "hit_rate": reuse.hit_rate,
            "contributors_lru_order": touched,
        })
    return out


def schedule_cases():
    def reqs(h, arrivals=None):
        arrivals = arrivals or list(range(len(h)))
        return [Request(f"r{i}", float(a), [], 0, x) for i, (x, a) in enumerate(zip(h, arrivals))]
    cases = []
    for h, arr, bs, lam, now in [([1.0, 0.0, 1.0, 0.0], None, 2, 0.0, 0.0),
                                 ([0.5] * 4, None, 2, 0.0, 0.0),
                                 ([0.9, 0.3, 0.3, 0.7, 0.1, 0.5], [5, 1, 2, 3, 4, 0], 2, 0.0, 0.0),
                                 ([0.9, 0.0], [1000.0, 0.0], 1, 0.01, 2000.0),
                                 ([0.2, 0.8, 0.8, 0.4, 0.6, 0.1, 0.9], None, 3, 0.0, 0.0)]:
        rs = reqs(h, arr)
        b = schedule(rs, bs, aging_lambda=lam, now_ms=now)
        cases.append({"hit": h, "arrival": [r.arrival_ms for r in rs], "ids": [r.id for r in rs],
                      "batch_size": bs, "aging": lam, "now": now,
                      "batches": [[r.id for r in x.requests] for x in b]})
    return cases


def _weights_digest(model) -> str:
    import hashlib
    h = hashlib.sha256(np.ascontiguousarray(model.embedding).tobytes())
    for l in model.layers:
        for w in (l.w_q, l.w_k, l.w_v, l.w_o):
            h.update(np.ascontiguousarray(w).tobytes())
    return h.hexdigest()


def _objs(items):
    out = np.empty(len(items), dtype=object)
    for i, x in enumerate(items):
        out[i] = np.asarray(x)
    return out


def model_case(name, cfg, w, ratio, n_extra, seed):
    """Scenario following studies._reuse_scenario / test_engine.scenario."""
    rng = np.random.default_rng(seed)
    model = init_model(cfg)
    pool = CachePool(cfg, HashParams(window_size=w))
    sources = []
    for s in range(2):
        src = rng.integers(0, cfg.vocab_size, int(rng.integers(20, 40))).tolist()
        st = model_forward(src, model)
        pool.insert(f"src{s}", src, st.k, st.v)
        sources.append(src)
    target = rng.integers(0, cfg.vocab_size, 5).tolist()
    target += sources[0][3:15]
    target += rng.integers(0, cfg.vocab_size, 4).tolist()
    target += sources[1][2:12]
    target += rng.integers(0, cfg.vocab_size, 3).tolist()
    reuse = pool.lookup(target)
    order = [e.request_id for e in sorted(pool.entries.values(), key=lambda e: -e.insert_seq)]
    n = len(target)
    src_entry = np.full(n, -1, np.int32)
    src_cand = np.full(n, -1, np.int32)
    for p, (e, c) in reuse.sources.items():
        src_entry[p] = order.index(e.request_id)
        src_cand[p] = c
    scfg = SelectionConfig(ratio=ratio, n_extra=n_extra)
    probe = 1 if cfg.num_layers >= 2 else 0
    qp, kt, vt, kp, vp = engine._perturbed_probe(model, target, reuse, probe)
    reused = sorted(reuse.sources)
    dk = engine._restrict_rows(kp - kt, set(reused))
    dv = engine._restrict_rows(vp - vt, set(reused))
    sel = selection.select_prefill(qp, kt + dk, dv, reused, scfg)
    pre = engine.prefill_with_selection(model, target, reuse, scfg)
    assert pre.selected == sel.indices
    session = pre.session
    decode = rng.integers(0, cfg.vocab_size, 6).tolist()
    chosen_log = []
    orig = session.recompute_positions

    def rec(positions):
        chosen_log.append(sorted(int(p) for p in positions))
        return orig(positions)
    session.recompute_positions = rec
    # record the decode-step q_t / scores of the first step too
    q_t0 = session.query_rows_probe(decode[0])
    dstep = selection.select_decode_step(q_t0, session.k[session.probe_layer],
                                         session.delta_v_probe(), pre.eligible, n_extra)
    ref = engine.ReuseSession(model, target)
    gen = engine.run_generation(session, ref, decode, n_extra)
    entry_k = [pool.entries[r].k for r in order]
    entry_v = [pool.entries[r].v for r in order]
    np.savez_compressed(
        os.path.join(HERE, f"golden_model_{name}.npz"),
        config=np.array([cfg.num_layers, cfg.num_heads, cfg.d_model, cfg.vocab_size, cfg.seed]),
        w=w, ratio=ratio, n_extra=n_extra,
        weights_sha256=np.array(_weights_digest(model)),
        **({"embedding": model.embedding,
            "layers": np.stack([np.stack([l.w_q, l.w_k, l.w_v, l.w_o]) for l in model.layers])}
           if name == "small" else {}),
        entry_tokens=_objs([pool.entries[r].tokens for r in order]),
        entry_k=_objs(entry_k), entry_v=_objs(entry_v),
        target=np.array(target), src_entry=src_entry, src_cand=src_cand,
        probe_q=qp, probe_k_true=kt, probe_v_true=vt, probe_k_pert=kp, probe_v_pert=vp,
        scores=sel.scores, selected=np.array(sel.indices, dtype=np.int64),
        eligible=np.array(sorted(pre.eligible), dtype=np.int64),
        prefill_hidden=session.prefill_states.hidden, prefill_k=session.prefill_states.k,
        prefill_v=session.prefill_states.v, prefill_head_out=session.prefill_states.head_out,
        decode_tokens=np.array(decode), decode_q_t0=q_t0, decode_scores0=dstep.scores,
        decode_chosen0=np.array(dstep.indices, dtype=np.int64),
        decode_recompute_counts=np.array(gen.recompute_counts),
        decode_chosen=_objs([np.array(c, dtype=np.int64) for c in chosen_log]),
        final_k=session.k, final_v=session.v,
    )


def main():
    rng = np.random.default_rng(20250317)
    doc = {"hashes": hash_cases(rng), "match": match_cases(rng),
           "lookup": lookup_cases(rng), "schedule": schedule_cases()}
    with open(os.path.join(HERE, "golden_match.json"), "w") as fh:
        json.dump(doc, fh, separators=(",", ":"))
    model_case("small", ModelConfig(num_layers=3, num_heads=2, d_model=16, vocab_size=256,
                                    seed=42), 4, 0.3, 3, 1)
    model_case("default", ModelConfig(num_layers=4, num_heads=4, d_model=64, vocab_size=4096,
                                      seed=7), 8, 0.2, 3, 2)
    model_case("wide", ModelConfig(num_layers=2, num_heads=2, d_model=128, vocab_size=512,
                                   seed=11), 8, 0.5, 2, 3)
    print("golden vectors written to", HERE)


if __name__ == "__main__":
    main()
