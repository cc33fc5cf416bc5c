"""Failure paths and non-default scaling modes through the CUDA product path,
against the oracle (the C restatement, pinned bitwise to the reference) and,
where it is built, the reference itself (oracle/_ref).

* Numerical trouble is a status, never an exception: a non-finite iterate, a
  collapsed or non-finite step, or more than 80 trials end the solve with
  kNumericalError (solver.hpp:417-420, 459-466, 385, 811-817). Pathological
  instances must give the reference's status in both modes, and parity mode
  its iteration count too.
* The reference's overflow guard (test_solver.cpp:507-515): magnitudes near
  DBL_MAX with no scaling must not produce a bogus Optimal.
* ScalingMode::kNone / kRuiz (scaling.hpp:16; test_solver.cpp:337-352): the
  scaling vectors bitwise equal to the reference's make_scaling, parity-mode
  solves bitwise, fast-mode solves optimal and passing the reference's
  termination check.
"""
from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as O
from paper_2311_12180_b200 import Mode, Solver, SolverParams, SolveStatus, generators, solve
from paper_2311_12180_b200.lp import CsrMatrix, GeneralFormLp, ScalingMode

pytestmark = pytest.mark.gpu


def kinds() -> list[str]:
    return ["oracle"] + (["ref"] if O.available("ref") else [])


def one_var(c: float, a: float, h: float, lo: float = 0.0, up: float = np.inf) -> GeneralFormLp:
    G = CsrMatrix.from_triplets(1, 1, [0], [0], [a])
    return GeneralFormLp(G, CsrMatrix.zero(0, 1), [c], [h], np.zeros(0), [lo], [up])


def dense_lp(Gd, h, Ad, b, c, lo, up) -> GeneralFormLp:
    n = len(c)

    def csr(d):
        d = np.asarray(d, float).reshape(-1, n)
        r, cc = np.nonzero(d)
        return CsrMatrix.from_triplets(d.shape[0], n, r, cc, d[r, cc])

    return GeneralFormLp(csr(Gd), csr(Ad), c, h, b, lo, up)


PATHOLOGICAL = {
    # test_solver.cpp:507-515: objective and rhs at 1e308, no scaling
    "overflow_guard": (lambda: one_var(1e308, 1.0, 1e308),
                       dict(scaling=ScalingMode.NONE, eps_optimal=1e-8, iteration_limit=1000)),
    # the same with the default preconditioner
    "overflow_scaled": (lambda: one_var(1e308, 1.0, 1e308), dict(eps_optimal=1e-8, iteration_limit=1000)),
    # a NaN in the matrix (GeneralFormLp::validate checks bounds and c only):
    # the first trial's iterate is non-finite -> kNumericalError (solver.hpp:417-420)
    "nan_matrix": (lambda: dense_lp([[1.0, np.nan]], [1.0], np.zeros((0, 2)), [], [1.0, 1.0], [0.0, 0.0],
                                    [10.0, 10.0]), dict(scaling=ScalingMode.NONE)),
    # an infinite matrix entry: the step size becomes NaN / the iterate non-finite
    "inf_matrix": (lambda: dense_lp([[1.0, np.inf]], [1.0], np.zeros((0, 2)), [], [1.0, 1.0], [0.0, 0.0],
                                    [10.0, 10.0]), dict(scaling=ScalingMode.NONE)),
    # tiny and huge magnitudes side by side (movement and interaction under/overflow)
    "mixed_magnitudes": (lambda: dense_lp([[1e-300, 1e300]], [1.0], [[1e300, 1.0]], [1e300], [1e-300, 1.0],
                                          [0.0, 0.0], [np.inf, np.inf]),
                         dict(scaling=ScalingMode.NONE, iteration_limit=2000)),
}


def extreme_lp(seed: int) -> tuple[GeneralFormLp, ScalingMode]:
    """Tiny LPs with magnitudes 10^U(-250, 250): overflowing movements and
    interactions, NaN step sizes and collapsing steps mid-solve."""
    rng = np.random.default_rng(seed)
    n, m1, m2 = int(rng.integers(1, 4)), int(rng.integers(0, 3)), int(rng.integers(1, 2))

    def e(size):
        return 10.0 ** rng.uniform(-250, 250, size=size) * rng.choice([-1.0, 1.0], size=size)

    Gd, Ad = e((m1, n)), e((m2, n))
    lp = dense_lp(Gd, e(m1), Ad, e(m2), e(n), np.zeros(n), np.full(n, np.inf))
    return lp, ScalingMode(int(rng.integers(0, 3)))


@pytest.mark.parametrize("mode", [Mode.FAST, Mode.PARITY])
def test_extreme_magnitudes_status_matches_reference(mode):
    """40 seeded extreme-magnitude instances: the same status as the
    reference (several end in kNumericalError after dozens of steps), and in
    parity mode the same iteration count."""
    seen = set()
    for seed in range(40):
        lp, scaling = extreme_lp(seed)
        p = SolverParams(mode=mode, scaling=scaling, iteration_limit=500, time_limit_seconds=60.0)
        r = solve(lp, p)
        o = O.solve(lp, p, kinds()[-1])
        assert r.status == o.status, (seed, r.status, o.status)
        if mode == Mode.PARITY:
            assert r.iterations == o.iterations, (seed, r.iterations, o.iterations)
        seen.add(r.status)
    assert SolveStatus.NUMERICAL_ERROR in seen


@pytest.mark.parametrize("name", sorted(PATHOLOGICAL))
@pytest.mark.parametrize("mode", [Mode.FAST, Mode.PARITY])
def test_pathological_status_matches_reference(name, mode):
    build, kw = PATHOLOGICAL[name]
    lp = build()
    p = SolverParams(mode=mode, time_limit_seconds=60.0, **kw)
    r = solve(lp, p)
    for kind in kinds():
        o = O.solve(lp, p, kind)
        assert r.status == o.status, (name, kind, r.status, o.status)
        if mode == Mode.PARITY:
            assert r.iterations == o.iterations, (name, kind)
    if name.startswith("overflow"):
        assert r.status != SolveStatus.OPTIMAL  # no bogus Optimal (test_solver.cpp:513-514)
    if name in ("nan_matrix", "inf_matrix"):
        assert r.status == SolveStatus.NUMERICAL_ERROR


def test_numerical_error_is_a_status_not_an_exception():
    """kNumericalError comes back through pdlp_solve as a status with the
    candidate point (solver.hpp:811-817): no exception crosses the ABI."""
    lp = PATHOLOGICAL["nan_matrix"][0]()
    with Solver(lp, SolverParams(scaling=ScalingMode.NONE)) as s:
        r = s.solve()
        assert r.status == SolveStatus.NUMERICAL_ERROR
        assert r.point.primal.shape == (2,) and r.point.dual.shape == (1,)
        r2 = s.solve()  # the handle stays usable
        assert r2.status == SolveStatus.NUMERICAL_ERROR


@pytest.mark.parametrize("scaling", [ScalingMode.NONE, ScalingMode.RUIZ, ScalingMode.RUIZ_POCK_CHAMBOLLE])
def test_scaling_modes_bitwise_and_optimal(scaling):
    lps = [generators.small_random_lp(n=12, m1=4, m2=3, seed=s) for s in (2025, 2026, 2027)]
    lps.append(generators.config("C1"))
    for i, lp in enumerate(lps):
        p = SolverParams(scaling=scaling, eps_optimal=1e-8 if i < 3 else 1e-4)
        d1, d2 = O.scaling(lp, p, kinds()[-1])
        with Solver(lp, p) as s:
            g1, g2 = s.scaling()
        assert np.array_equal(g1, d1) and np.array_equal(g2, d2), (scaling, i)
        par = solve(lp, SolverParams(scaling=scaling, mode=Mode.PARITY, eps_optimal=p.eps_optimal))
        ora = O.solve(lp, p, "oracle")
        assert par.status == ora.status and par.iterations == ora.iterations, (scaling, i)
        assert np.array_equal(par.point.primal, ora.point.primal) and np.array_equal(par.point.dual, ora.point.dual)
        fast = solve(lp, p)
        assert fast.status == SolveStatus.OPTIMAL == ora.status, (scaling, i)
        chk = O.check_termination(lp, fast.point.primal, fast.point.dual, p.eps_optimal, kinds()[-1])
        assert chk["terminated"], (scaling, i, chk)
