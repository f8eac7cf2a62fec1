"""Generate F4 comparison-strategy goldens by running the REFERENCE here.

    python tests/golden/make_golden_select.py [/root/reference/pkg/src]

golden_strategies.npz: for random reuse instances (q, k, v fresh; dk, dv the
cached-minus-fresh increments on the reused rows, zero elsewhere; multi-head,
causal) the reference's select_baseline (selection.py:133-186) indices and
scores for MAGNITUDE, POSITIONAL, RANDOM (seeded) and IDEAL, plus
ATTENTION_WEIGHTED for cross-checking.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = next((a for a in sys.argv[1:] if not a.startswith("--")), "/root/reference/pkg/src")
sys.path.insert(0, REF)
os.environ["KVLAB_MATCH_BACKEND"] = "pure"

from kvlab.selection import SelectionConfig, Strategy, select_baseline  # noqa: E402

STRATS = ["magnitude", "positional", "random", "ideal", "attention_weighted"]


def main():
    rng = np.random.default_rng(21)
    out = {}
    cases = 12
    for c in range(cases):
        H = int(rng.choice([1, 2, 4]))
        n = int(rng.integers(6, 48))
        d = int(rng.choice([4, 8, 16]))
        q, k, v = (rng.normal(size=(H, n, d)) for _ in range(3))
        reused = sorted(rng.choice(n, size=int(rng.integers(1, n)), replace=False).tolist())
        mask = np.zeros(n, bool)
        mask[reused] = True
        dk = rng.normal(size=(H, n, d)) * 0.3 * mask[None, :, None]
        dv = rng.normal(size=(H, n, d)) * 0.3 * mask[None, :, None]
        ratio = float(rng.choice([0.2, 0.3, 0.5, 1.0]))
        seed = int(rng.integers(0, 1000))
        cfg = SelectionConfig(ratio=ratio, seed=seed)
        for name, x in (("q", q), ("k", k), ("v", v), ("dk", dk), ("dv", dv)):
            out[f"c{c}_{name}"] = x
        out[f"c{c}_reused"] = np.array(reused)
        out[f"c{c}_meta"] = np.array([ratio, seed])
        for s in STRATS:
            res = select_baseline(Strategy(s), q, k, v, dk, dv, reused, cfg)
            out[f"c{c}_{s}_idx"] = np.array(res.indices, dtype=np.int64)
            out[f"c{c}_{s}_scores"] = np.asarray(res.scores, float)
    out["n_cases"] = np.array(cases)
    np.savez_compressed(os.path.join(HERE, "golden_strategies.npz"), **out)
    print("cases", cases)


if __name__ == "__main__":
    main()


def oracle_mode_cases():
    """golden_oracle_mode.npz: reference prefill_with_selection in ORACLE mode
    (engine.py:245-285) for every strategy on one small reuse scenario, with
    the scenario inputs the restatement needs."""
    from kvlab import engine
    from kvlab.matching import HashParams
    from kvlab.model import ModelConfig, init_model, model_forward
    from kvlab.pool import CachePool
    from kvlab.selection import SelectionMode
    cfg = ModelConfig(num_layers=3, num_heads=2, d_model=16, vocab_size=256, seed=4)
    model = init_model(cfg)
    rng = np.random.default_rng(8)
    pool = CachePool(cfg, HashParams(window_size=4))
    srcs = []
    for s in range(2):
        src = rng.integers(0, 256, int(rng.integers(25, 40))).tolist()
        st = model_forward(src, model)
        pool.insert(f"s{s}", src, st.k, st.v)
        srcs.append(src)
    target = (rng.integers(0, 256, 4).tolist() + srcs[0][2:20] + rng.integers(0, 256, 3).tolist()
              + srcs[1][4:16] + rng.integers(0, 256, 2).tolist())
    reuse = pool.lookup(target)
    ref = model_forward(target, model)
    order = [e.request_id for e in sorted(pool.entries.values(), key=lambda e: -e.insert_seq)]
    n = len(target)
    src_entry = np.full(n, -1, np.int32)
    src_cand = np.full(n, -1, np.int32)
    for p, (e, c) in reuse.sources.items():
        src_entry[p] = order.index(e.request_id)
        src_cand[p] = c
    out = {"target": np.array(target), "src_entry": src_entry, "src_cand": src_cand,
           "ref_k": ref.k, "ref_v": ref.v,
           "config": np.array([cfg.num_layers, cfg.num_heads, cfg.d_model, cfg.vocab_size,
                               cfg.seed])}
    for i, r in enumerate(order):
        out[f"entry_tokens_{i}"] = pool.entries[r].tokens
        out[f"entry_k_{i}"] = pool.entries[r].k
        out[f"entry_v_{i}"] = pool.entries[r].v
    out["n_entries"] = np.array(len(order))
    for s in STRATS:
        scfg = SelectionConfig(ratio=0.3, mode=SelectionMode.ORACLE, strategy=Strategy(s), seed=5)
        res = engine.prefill_with_selection(model, target, reuse, scfg, ref_states=ref)
        for layer, st in enumerate(res.recompute_sets):
            out[f"{s}_set{layer}"] = np.array(sorted(st), dtype=np.int64)
        out[f"{s}_hidden"] = res.session.prefill_states.hidden
    np.savez_compressed(os.path.join(HERE, "golden_oracle_mode.npz"), **out)
    print("oracle-mode golden written")


if __name__ == "__main__" and "--oracle-mode" in sys.argv:
    oracle_mode_cases()


def serving_cases():
    """golden_serving.json: reference run_simulation (simulate.py:140-215) on
    generated traces - per request TTFT, completion, hit rate - for the
    cache-aware and FCFS schedulers and the adaptive / fixed matchers."""
    import json as _json
    from kvlab.model import ModelConfig
    from kvlab.simulate import MatcherKind, SchedulerKind, SimConfig, run_simulation
    from kvlab.trace import generate_trace
    out = []
    for sched in (SchedulerKind.CACHE_AWARE, SchedulerKind.FCFS):
        for matcher in (MatcherKind.ADAPTIVE, MatcherKind.FIXED):
            for overlap, gap in ((0.8, 20.0), (0.5, 60.0)):
                trace = generate_trace(num_requests=10, seed=3, vocab_size=512, overlap=overlap,
                                       arrival_gap_ms=gap, decode_steps=4)
                cfg = SimConfig(model=ModelConfig(num_layers=2, num_heads=2, d_model=16,
                                                  vocab_size=512, seed=1),
                                batch_size=3, scheduler=sched, matcher=matcher, window_size=4,
                                chunk_size=8)
                rep = run_simulation(trace, cfg)
                out.append({
                    "scheduler": sched.value, "matcher": matcher.value, "overlap": overlap,
                    "gap": gap,
                    "trace": [{"id": r.id, "arrival_ms": r.arrival_ms, "tokens": r.tokens,
                               "decode_steps": r.decode_steps} for r in trace],
                    "requests": [{"id": m.id, "ttft_ms": m.ttft_ms,
                                  "completion_ms": m.completion_ms, "hit_rate": m.hit_rate}
                                 for m in rep.requests],
                    "aggregate": {k: rep.aggregate[k] for k in ("mean_ttft_ms", "p50_ttft_ms",
                                                                "makespan_ms")},
                })
    with open(os.path.join(HERE, "golden_serving.json"), "w") as fh:
        _json.dump(out, fh)
    print("serving golden:", len(out))


if __name__ == "__main__" and "--serving" in sys.argv:
    serving_cases()
