"""NEXT-4: the paper's analytical latency model, attention terms,
with coefficients fitted to this build's kernels on B200.

PAPER.md Appendix A. Symbols: h hidden size per GPU
(h = n * s after tensor parallelism), n heads, s head size, B batch size, l_i
the length of request i, t = sum_i l_i, t2 = sum_i l_i^2, b the block size of
the attention kernel.

  prefill attention, one layer:  T2 = C2 * 3 h t2 / b
  decode attention, one layer:  T4 = C5 * 3 h t

The paper folds fixed overheads into C3 (whole prefill) and C4 (decode
GEMMs). Here only the attention kernels are modelled, so `fit` can add a
per-launch intercept (reported separately) — the launch + prologue cost a
persistent B200 kernel pays that the paper's A100 profile hides in C3/C4.

For decode, l_i is the number of tokens attended in the step: the cached c_i
plus the token appended in that step (reading R9 of DESIGN.md).
b: the paper's FlashAttention block size; our prefill re-reads K/V once per
128-row query tile, so B_PREFILL = 128 here (the coefficient absorbs the choice).

Pure host arithmetic (numpy); no GPU, no oracle.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

B_PREFILL = 128


def prefill_feature(lens, n: int, s: int, b: int = B_PREFILL) -> float:
    """3 h t2 / b for one layer of prefill attention."""
    t2 = float(sum(int(l) * int(l) for l in lens))
    return 3.0 * n * s * t2 / b


def prefill_linear_feature(lens, n: int, s: int) -> float:
    """2 h t: the 2 s l term of the exact count "2 s l + 3 s l (l / b)" that
    the paper drops (T2 keeps only the quadratic part); kept in the `full` fit."""
    return 2.0 * n * s * float(sum(int(l) for l in lens))


def decode_feature(attended_lens, n: int, s: int) -> float:
    """3 h t for one layer of decode attention; attended_lens = c_i + 1."""
    t = float(sum(int(l) for l in attended_lens))
    return 3.0 * n * s * t


@dataclass
class Fit:
    coef: list           # one coefficient per feature (C2 or C5 first), seconds per unit
    intercept: float     # seconds per launch (0 when fitted without one)
    r2: float
    max_rel_err: float   # max_i |pred_i - y_i| / y_i over the fitted points
    points: int

    def predict(self, x):
        X = np.asarray(x, dtype=np.float64)
        X = X[:, None] if X.ndim == 1 else X
        return X @ np.asarray(self.coef) + self.intercept

    def as_dict(self):
        return {"coef": self.coef, "intercept_s": self.intercept, "r2": self.r2, "max_rel_err": self.max_rel_err,
                "points": self.points}


def fit(x, y, intercept: bool = True) -> Fit:
    """Least squares y ~ x . C (+ c0), the "profiling and interpolation" of P:682/P:704.
    x: [points] (one feature) or [points][features]. Relative weighting (each point
    divided by its y) so that short launches count as much as long ones."""
    X = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    X = X[:, None] if X.ndim == 1 else X
    if X.ndim != 2 or y.ndim != 1 or X.shape[0] != y.shape[0]:
        raise ValueError("need x [points] or [points][features] and y [points]")
    if X.shape[0] < X.shape[1] + (1 if intercept else 0):
        raise ValueError("not enough points for the number of coefficients")
    if np.any(y <= 0):
        raise ValueError("latencies must be positive")
    A = np.concatenate([X, np.ones((len(y), 1))], axis=1) if intercept else X
    w = 1.0 / y
    sol, *_ = np.linalg.lstsq(A * w[:, None], y * w, rcond=None)
    coef = [float(c) for c in sol[:X.shape[1]]]
    c0 = float(sol[-1]) if intercept else 0.0
    pred = X @ np.asarray(coef) + c0
    ss_res = float(np.sum((y - pred) ** 2))
    ss_tot = float(np.sum((y - y.mean()) ** 2))
    r2 = 1.0 - ss_res / ss_tot if ss_tot > 0 else 1.0
    return Fit(coef, c0, r2, float(np.max(np.abs(pred - y) / y)), len(y))
