"""pdhg_raw_step (solver.hpp:335-358) on the GPU: one plain PDHG step with
explicit extrapolation on the unscaled saddle problem, through the C-ABI
(pdlp_pdhg_raw_step). The reference's own known answers
(test_solver.cpp:33-61) plus seeded LPs against the oracle and the reference
compiled in place: parity mode bitwise, fast mode within 1e-13."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as O
from paper_2311_12180_b200 import Mode, Solver, SolverParams, generators
from paper_2311_12180_b200.lp import CsrMatrix, GeneralFormLp

pytestmark = pytest.mark.gpu


def csr(rows, cols, dense):
    dense = np.asarray(dense, dtype=np.float64).reshape(rows, cols)
    off, col, val = [0], [], []
    for r in range(rows):
        for c in range(cols):
            if dense[r, c] != 0.0:
                col.append(c)
                val.append(dense[r, c])
        off.append(len(col))
    return CsrMatrix(rows, cols, np.array(off, np.int64), np.array(col, np.int64), np.array(val))


def empty(cols):
    return CsrMatrix(0, cols, np.zeros(1, np.int64), np.zeros(0, np.int64), np.zeros(0))


def origin_lp():
    # LpBuilder(2).objective({0, 0}).geq({1, 1}, 0).free_variable(0).free_variable(1)
    return GeneralFormLp(csr(1, 2, [1.0, 1.0]), empty(2), np.zeros(2), np.zeros(1), np.zeros(0),
                         np.full(2, -np.inf), np.full(2, np.inf))


def one_var_lp():
    # min x s.t. x >= 1, x in [0, 10] (test_solver.cpp:18-21)
    return GeneralFormLp(csr(1, 1, [1.0]), empty(1), np.ones(1), np.ones(1), np.zeros(0), np.zeros(1),
                         np.full(1, 10.0))


@pytest.mark.parametrize("mode", [Mode.PARITY, Mode.FAST])
def test_known_answers(mode):
    """test_solver.cpp:33-61: the origin is a fixed point when c and q vanish;
    the one-variable hand trace gives y' = 0.5; a saddle point is fixed."""
    with Solver(origin_lp(), SolverParams(mode=mode)) as s:
        x, y = s.pdhg_raw_step(np.zeros(2), np.zeros(1), 0.7, 0.3)
        assert x.tolist() == [0.0, 0.0] and y.tolist() == [0.0]
    with Solver(one_var_lp(), SolverParams(mode=mode)) as s:
        x, y = s.pdhg_raw_step(np.zeros(1), np.zeros(1), 0.5, 0.5)
        assert x.tolist() == [0.0] and y.tolist() == [0.5]
        x, y = s.pdhg_raw_step(np.ones(1), np.ones(1), 0.4, 0.9)
        assert x.tolist() == [1.0] and y.tolist() == [1.0]


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_seeded_lps_against_oracle_and_reference(seed):
    lp = generators.random_lp(400, 300, 1200, 6, seed=seed)
    rng = np.random.default_rng(seed)
    x = rng.uniform(-1.0, 3.0, lp.num_variables)
    y = rng.uniform(-2.0, 2.0, lp.num_constraints)
    want = O.pdhg_raw_step(lp, x, y, 0.3, 0.7, "oracle")
    if O.available("ref"):  # the oracle is pinned to the reference here too
        ref = O.pdhg_raw_step(lp, x, y, 0.3, 0.7, "ref")
        assert np.array_equal(ref[0], want[0]) and np.array_equal(ref[1], want[1])
    with Solver(lp, SolverParams(mode=Mode.PARITY)) as s:
        got = s.pdhg_raw_step(x, y, 0.3, 0.7)
    assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])
    with Solver(lp, SolverParams()) as s:
        fast = s.pdhg_raw_step(x, y, 0.3, 0.7)
    for a, b in zip(fast, want):
        assert np.max(np.abs(a - b)) <= 1e-13 * max(1.0, np.max(np.abs(b)))


def test_errors():
    with Solver(one_var_lp(), SolverParams()) as s:
        with pytest.raises(ValueError, match="dimension mismatch"):
            s.pdhg_raw_step(np.zeros(2), np.zeros(1), 0.5, 0.5)
        with pytest.raises(ValueError, match="positive and finite"):
            s.pdhg_raw_step(np.zeros(1), np.zeros(1), 0.0, 0.5)
