"""Seeded synthetic LP generators for the BASELINE.json configurations.

Recipes follow SURVEY.md §8(d) (the reference ships no generator at these
sizes; its small-instance pattern is test_oracle::random_feasible_lp,
tests/oracle/lp_builder.hpp:83-132: an interior point x0, b = A x0,
h = G x0 - U(0, 2), boxes [0, 10], coefficients U(-3, 3) with 0 -> 1,
c ~ U(-3, 3)). Column patterns are sampled without replacement, so the CSR
never has duplicates for from_triplets to fold.

  C1 random          random_lp(5000, 5000, 20000, 5, seed=20261001)
  C2 transportation  transport_lp(1000, 1000, seed=20261002)
  C3 multicommodity  multicommodity_lp(20000, 100000, 50, seed=20261003)
  C4 random          random_lp(10**7, 10**7, 4 * 10**7, 5, seed=20261004)
  C5 staircase       staircase_lp(64, 2_500_000, 625_000, 625_000, seed=20261005)
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


def multicommodity_lp(nodes: int = 20000, arcs: int = 100000, commodities: int = 50,
                      seed: int = SEEDS["C3"], gamma: float = 2.1) -> GeneralFormLp:
    """Multicommodity flow (C3): a Chung-Lu power-law digraph
    (expected degree ~ (i+1)^(-1/(gamma-1))), variable x[k, a] = flow of
    commodity k on arc a (column k * arcs + a). Rows, inequalities first:
      capacity   per arc a:        -sum_k x[k, a] >= -cap_a          (length K)
      budget     per commodity k:  -sum_a w_a x[k, a] >= -B_k        (length arcs)
      conservation per (k, v):     sum_out x - sum_in x = b_kv      (length deg v)
    A strictly interior flow x0 ~ U(0.5, 1.5) fixes b = A x0, cap = 1.2 load,
    B = 1.2 cost(x0), so the LP is feasible; costs w ~ U{1..20} keep it bounded.
    Row lengths run from 1 to `arcs` (merge-path / CHUNK tiles)."""
    rng = np.random.default_rng(seed)
    V, E, K = nodes, arcs, commodities
    w = (np.arange(V) + 1.0) ** (-1.0 / (gamma - 1.0))
    p = w / w.sum()
    src = rng.choice(V, size=E, p=p)
    dst = rng.choice(V, size=E, p=p)
    loop = src == dst
    while loop.any():
        dst[loop] = rng.choice(V, size=int(loop.sum()), p=p)
        loop = src == dst
    cost = rng.integers(1, 21, size=E).astype(np.float64)
    x0 = rng.uniform(0.5, 1.5, size=(K, E))
    n = K * E
    # capacity rows: row a has columns k*E + a, k = 0..K-1 (ascending)
    cap_off = np.arange(E + 1, dtype=np.int64) * K
    cap_col = (np.arange(K, dtype=np.int64)[None, :] * E + np.arange(E)[:, None]).reshape(-1)
    cap_val = -np.ones(E * K)
    cap = 1.2 * x0.sum(axis=0)
    # budget rows: row k has columns k*E .. k*E + E - 1
    bud_off = np.arange(K + 1, dtype=np.int64) * E
    bud_col = np.arange(n, dtype=np.int64)
    bud_val = -np.tile(cost, K)
    budget = 1.2 * (x0 * cost[None, :]).sum(axis=1)
    # conservation rows (k, v): arcs leaving v (+1) and entering v (-1), column-sorted
    node = np.concatenate([src, dst])
    arc = np.concatenate([np.arange(E), np.arange(E)])
    sign = np.concatenate([np.ones(E), -np.ones(E)])
    order = np.lexsort((arc, node))
    node, arc, sign = node[order], arc[order], sign[order]
    deg = np.bincount(node, minlength=V)
    base_off = np.zeros(V + 1, np.int64)
    np.cumsum(deg, out=base_off[1:])
    nnz_c = 2 * E
    con_off = (np.arange(K, dtype=np.int64)[:, None] * nnz_c + base_off[None, :-1]).reshape(-1)
    con_off = np.concatenate([con_off, [K * nnz_c]])
    con_col = (np.arange(K, dtype=np.int64)[:, None] * E + arc[None, :]).reshape(-1)
    con_val = np.tile(sign, K)
    # b = A x0, per commodity: node balance of x0[k]
    bal = np.zeros((K, V))
    for k in range(K):
        bal[k] = np.bincount(src, weights=x0[k], minlength=V) - np.bincount(dst, weights=x0[k], minlength=V)
    g_off = np.concatenate([cap_off, cap_off[-1] + bud_off[1:]])
    G = CsrMatrix(E + K, n, g_off, np.concatenate([cap_col, bud_col]).astype(np.int32),
                  np.concatenate([cap_val, bud_val]))
    A = CsrMatrix(K * V, n, con_off, con_col.astype(np.int32), con_val)
    c = np.tile(cost, K)
    return GeneralFormLp(G, A, c, np.concatenate([-cap, -budget]), bal.reshape(-1), np.zeros(n),
                         np.full(n, np.inf))


def staircase_lp(stages: int = 64, n_stage: int = 2_500_000, m1_stage: int = 625_000,
                 m2_stage: int = 625_000, per_col: int = 6, seed: int = SEEDS["C5"],
                 box: float = 10.0) -> GeneralFormLp:
    """Staircase LP (C5): T stages of n_t variables and
    m_t = m1_t + m2_t rows; the intra-stage block has `per_col` nonzeros per
    column (one random pattern shared by every stage, fresh values per stage);
    equality row i of stage t > 0 also carries +1 on variable i of stage t - 1
    (the state coupling). Rows are ordered inequalities of all stages, then
    equalities of all stages; an interior x0 ~ U(1, 6) fixes b = A x0 and
    h = G x0 - U(0, 2). Column blocks are stage-contiguous, so a row shard on
    stage boundaries touches only its own columns plus the previous stage's."""
    rng = np.random.default_rng(seed)
    T, nt, m1t, m2t = stages, n_stage, m1_stage, m2_stage
    mt = m1t + m2t
    rows = rng.integers(0, mt, size=(nt, per_col), dtype=np.int64)
    rows.sort(axis=1)
    while True:
        dup = (np.diff(rows, axis=1) == 0).any(axis=1)
        if not dup.any():
            break
        idx = np.nonzero(dup)[0]
        fresh = rng.integers(0, mt, size=(idx.size, per_col), dtype=np.int64)
        fresh.sort(axis=1)
        rows[idx] = fresh
    off, col, _ = _csr_from_columns(rows, np.zeros((nt, per_col)), mt, nt, per_col)
    lens = np.diff(off)
    nnz_t = int(off[-1])
    n = T * nt
    x0 = rng.uniform(1.0, 6.0, size=n)
    c = rng.uniform(-3.0, 3.0, size=n)
    g_parts, a_parts = [], []
    g_rhs, a_rhs = [], []
    for t in range(T):
        vals = rng.uniform(-3.0, 3.0, size=nnz_t)
        vals[vals == 0.0] = 1.0
        cols_t = col.astype(np.int64) + t * nt
        rid = np.repeat(np.arange(mt), lens)
        act = np.bincount(rid, weights=vals * x0[cols_t], minlength=mt)
        kg = int(off[m1t])
        g_parts.append((lens[:m1t], cols_t[:kg], vals[:kg]))
        g_rhs.append(act[:m1t] - rng.uniform(0.0, 2.0, size=m1t))
        a_len = lens[m1t:].copy()
        a_col = cols_t[kg:]
        a_val = vals[kg:]
        if t > 0:  # coupling +1 on state variable i of stage t-1, which precedes the row's own columns
            couple = np.arange(m2t, dtype=np.int64) + (t - 1) * nt
            starts = np.concatenate([[0], np.cumsum(a_len)[:-1]])
            a_col = np.insert(a_col, starts, couple)
            a_val = np.insert(a_val, starts, 1.0)
            a_len = a_len + 1
            act_a = act[m1t:] + x0[couple]
        else:
            act_a = act[m1t:]
        a_parts.append((a_len, a_col, a_val))
        a_rhs.append(act_a)

    def stack(parts, m):
        lens_all = np.concatenate([p[0] for p in parts])
        o = np.zeros(m + 1, np.int64)
        np.cumsum(lens_all, out=o[1:])
        return o, np.concatenate([p[1] for p in parts]).astype(np.int32), np.concatenate([p[2] for p in parts])

    go, gc, gv = stack(g_parts, T * m1t)
    ao, ac, av = stack(a_parts, T * m2t)
    G = CsrMatrix(T * m1t, n, go, gc, gv)
    A = CsrMatrix(T * m2t, n, ao, ac, av)
    return GeneralFormLp(G, A, c, np.concatenate(g_rhs), np.concatenate(a_rhs), np.zeros(n), np.full(n, box))


def config(name: str) -> GeneralFormLp:
    if name == "C1":
        return random_lp(5000, 5000, 20000, 5, SEEDS["C1"])
    if name == "C2":
        return transport_lp(1000, 1000, SEEDS["C2"])
    if name == "C3":
        return multicommodity_lp(20000, 100000, 50, SEEDS["C3"])
    if name == "C4":
        return random_lp(10_000_000, 10_000_000, 40_000_000, 5, SEEDS["C4"])
    if name == "C5":
        return staircase_lp(64, 2_500_000, 625_000, 625_000, 6, SEEDS["C5"])
    raise KeyError(name)
