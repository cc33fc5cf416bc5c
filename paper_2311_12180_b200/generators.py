"""Seeded synthetic LP generators for the BASELINE.json configurations.

Recipes follow SURVEY.md §8(d) (the reference ships no generator at these
sizes; its small-instance pattern is test_oracle::random_feasible_lp,
tests/oracle/lp_builder.hpp:83-132: an interior point x0, b = A x0,
h = G x0 - U(0, 2), boxes [0, 10], coefficients U(-3, 3) with 0 -> 1,
c ~ U(-3, 3)). Column patterns are sampled without replacement, so the CSR
never has duplicates for from_triplets to fold.

  C1 random          random_lp(5000, 5000, 20000, 5, seed=20261001)
  C2 transportation  transport_lp(1000, 1000, seed=20261002)
  C4 random          random_lp(10**7, 10**7, 4 * 10**7, 5, seed=20261004)
"""
from __future__ import annotations

import numpy as np

from .lp import CsrMatrix, GeneralFormLp

SEEDS = {"C1": 20261001, "C2": 20261002, "C3": 20261003, "C4": 20261004, "C5": 20261005}


def _csr_from_columns(rows: np.ndarray, vals: np.ndarray, m: int, n: int, k: int):
    """rows/vals are (n, k) per-column patterns; returns CSR of the m x n matrix."""
    cols = np.repeat(np.arange(n, dtype=np.int64), k)
    r = rows.reshape(-1)
    order = np.argsort(r, kind="stable")  # keeps columns ascending within a row
    r_sorted = r[order]
    counts = np.bincount(r_sorted, minlength=m)
    off = np.zeros(m + 1, np.int64)
    np.cumsum(counts, out=off[1:])
    return off, cols[order].astype(np.int32), vals.reshape(-1)[order]


def random_lp(m1: int, m2: int, n: int, per_col: int = 5, seed: int = SEEDS["C1"],
              box: float = 10.0) -> GeneralFormLp:
    """Random sparse feasible LP (C1/C4 recipe): every column has `per_col`
    distinct rows; rows [0, m1) are inequalities G x >= h, the rest A x = b."""
    rng = np.random.default_rng(seed)
    m = m1 + m2
    rows = rng.integers(0, m, size=(n, per_col), dtype=np.int64)
    rows.sort(axis=1)
    while True:  # resample columns with repeated rows (without replacement)
        dup = (np.diff(rows, axis=1) == 0).any(axis=1)
        if not dup.any():
            break
        idx = np.nonzero(dup)[0]
        fresh = rng.integers(0, m, size=(idx.size, per_col), dtype=np.int64)
        fresh.sort(axis=1)
        rows[idx] = fresh
    vals = rng.uniform(-3.0, 3.0, size=(n, per_col))
    vals[vals == 0.0] = 1.0
    off, col, val = _csr_from_columns(rows, vals, m, n, per_col)
    x0 = rng.uniform(1.0, 6.0, size=n)
    # row activities K x0 (sequential per row, like spmv)
    rid = np.repeat(np.arange(m), np.diff(off))
    act = np.bincount(rid, weights=val * x0[col], minlength=m)
    slack = rng.uniform(0.0, 2.0, size=m1)
    h = act[:m1] - slack
    b = act[m1:]
    c = rng.uniform(-3.0, 3.0, size=n)
    nnz_g = int(off[m1])
    G = CsrMatrix(m1, n, off[: m1 + 1].copy(), col[:nnz_g], val[:nnz_g])
    A = CsrMatrix(m2, n, off[m1:] - nnz_g, col[nnz_g:], val[nnz_g:])
    return GeneralFormLp(G, A, c, h, b, np.zeros(n), np.full(n, box))


def transport_lp(supplies: int = 1000, demands: int = 1000, seed: int = SEEDS["C2"],
                 assignment: bool = False) -> GeneralFormLp:
    """Balanced transportation LP (C2): x_ij >= 0, sum_j x_ij = s_i,
    sum_i x_ij = d_j; integer costs U{1..100}, s, d ~ U{10..100} rebalanced so
    sum s = sum d (assignment: s = d = 1). Variable (i, j) is column i*D + j."""
    rng = np.random.default_rng(seed)
    S, D = supplies, demands
    n = S * D
    cost = rng.integers(1, 101, size=n).astype(np.float64)
    if assignment:
        s = np.ones(S)
        d = np.ones(D)
    else:
        s = rng.integers(10, 101, size=S).astype(np.float64)
        d = rng.integers(10, 101, size=D).astype(np.float64)
        diff = s.sum() - d.sum()
        if diff > 0:
            d[np.argmin(d)] += diff
        elif diff < 0:
            s[np.argmin(s)] += -diff
    # supply rows: contiguous column blocks; demand rows: stride-D columns
    sup_off = np.arange(S + 1, dtype=np.int64) * D
    sup_col = np.arange(n, dtype=np.int32)
    dem_off = S * D + np.arange(D + 1, dtype=np.int64) * S
    dem_col = (np.arange(S, dtype=np.int32)[None, :] * D + np.arange(D, dtype=np.int32)[:, None]).reshape(-1)
    off = np.concatenate([sup_off, dem_off[1:]])
    col = np.concatenate([sup_col, dem_col])
    A = CsrMatrix(S + D, n, off, col, np.ones(2 * n))
    G = CsrMatrix(0, n, np.zeros(1, np.int64), np.zeros(0, np.int32), np.zeros(0))
    return GeneralFormLp(G, A, cost, np.zeros(0), np.concatenate([s, d]), np.zeros(n), np.full(n, np.inf))


def small_random_lp(n: int, m1: int, m2: int, seed: int, density: float = 0.6,
                    box: float = 10.0) -> GeneralFormLp:
    """Dense-ish tiny feasible LP in the style of random_feasible_lp
    (lp_builder.hpp:83-132) for parity tests."""
    rng = np.random.default_rng(seed)
    x0 = rng.uniform(0.0, 1.0, size=n) * box * 0.5 + box * 0.1
    c = rng.uniform(-3.0, 3.0, size=n)

    def block(rows: int):
        mask = rng.uniform(size=(rows, n)) < density
        vals = rng.uniform(-3.0, 3.0, size=(rows, n))
        vals[vals == 0.0] = 1.0
        empty = ~mask.any(axis=1)
        mask[empty, rng.integers(0, n, size=empty.sum())] = True
        dense = np.where(mask, vals, 0.0)
        return dense

    Gd = block(m1)
    Ad = block(m2)
    h = Gd @ x0 - rng.uniform(0.0, 2.0, size=m1)
    b = Ad @ x0

    def csr(d):
        r, cc = np.nonzero(d)
        return CsrMatrix.from_triplets(d.shape[0], n, r, cc, d[r, cc])

    return GeneralFormLp(csr(Gd), csr(Ad), c, h, b, np.zeros(n), np.full(n, box))


def config(name: str) -> GeneralFormLp:
    if name == "C1":
        return random_lp(5000, 5000, 20000, 5, SEEDS["C1"])
    if name == "C2":
        return transport_lp(1000, 1000, SEEDS["C2"])
    if name == "C4":
        return random_lp(10_000_000, 10_000_000, 40_000_000, 5, SEEDS["C4"])
    raise KeyError(name)
