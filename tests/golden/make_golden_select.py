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
REF = sys.argv[1] if len(sys.argv) > 1 else "/root/reference/pkg/src"
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
