"""Tolerance helpers shared by the GPU parity tests (SURVEY.md 8c contract).

* integer outputs: bit-exact (asserted directly in the tests);
* scores / alpha: max |gpu - oracle| <= SCORE_TOL * max|oracle| (bf16 operands,
  fp32 accumulation, oracle on the same bf16-rounded inputs in float64);
* hidden rows / attention outputs: relative Frobenius error <= HIDDEN_TOL;
* selected sets: may differ only at indices whose oracle score lies within
  the score tolerance band around the B-th score (ties).
"""
import numpy as np

SCORE_TOL = 1.5e-2
HIDDEN_TOL = 2e-2


def bf16(x):
    """Round float64 arrays through bf16 (round-to-nearest-even)."""
    import torch
    return torch.as_tensor(np.asarray(x, dtype=np.float32)).to(torch.bfloat16).double().numpy()


def assert_scores_close(got, want, tol=SCORE_TOL):
    got, want = np.asarray(got, float), np.asarray(want, float)
    scale = max(np.abs(want).max(), 1e-30)
    err = np.abs(got - want).max() / scale
    assert err <= tol, f"score error {err:.3e} > {tol}"


def assert_rel_fro(got, want, tol=HIDDEN_TOL):
    got, want = np.asarray(got, float), np.asarray(want, float)
    err = np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-30)
    assert err <= tol, f"relative Frobenius error {err:.3e} > {tol}"


def assert_selection_tie_band(got, want, oracle_scores, budget, tol=SCORE_TOL):
    got, want = set(int(i) for i in got), set(int(i) for i in want)
    assert len(got) == len(want) == budget
    if got == want:
        return
    s = np.asarray(oracle_scores, float)
    band = tol * max(np.abs(s).max(), 1e-30)
    kth = sorted((s[i] for i in want), reverse=False)[0] if want else 0.0
    for i in got ^ want:
        assert abs(s[i] - kth) <= 2 * band, \
            f"index {i} (score {s[i]:.4e}) differs outside the tie band around {kth:.4e}"
