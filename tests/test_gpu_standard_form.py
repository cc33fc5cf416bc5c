"""The standard-form theory harness on the B200 (standard_form.py /
csrc/standard_form.cu) against the reference's standard_form.hpp, through the
golden traces it produced (tests/golden/make_golden_standard.py).

Bars: parity mode bitwise (spectral norm, KKT error, P_s norm, every epoch's
start KKT and length, the counters, the last epoch start and the first 200
recorded iterates); fast mode within fp64 tolerances, and the theorem
properties of acceptance criterion 5 (acceptance_main.cpp:232-331): KKT at
the n-th restart <= 0.5^n of the first, and the P_s distance to z* not growing
inside an epoch."""
from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

from paper_2311_12180_b200 import abi
from paper_2311_12180_b200.lp import CsrMatrix, PrimalDualPoint
from paper_2311_12180_b200.standard_form import (StandardFormLp, StandardPdhgOptions, kkt_error_standard,
                                                 p_s_norm_squared, restarted_pdhg_standard, spectral_norm)

pytestmark = pytest.mark.gpu
G = np.load(Path(__file__).resolve().parent / "golden" / "standard_golden.npz")
NAMES = ["f0", "f1", "f2", "f3", "f4", "r30x60", "r200x500"]


def instance(name: str) -> StandardFormLp:
    off, col, val = G[f"{name}/off"], G[f"{name}/col"], G[f"{name}/val"]
    m, n = len(off) - 1, len(G[f"{name}/c"])
    return StandardFormLp(CsrMatrix(m, n, off, col, val), G[f"{name}/b"], G[f"{name}/c"])


def options(name: str, parity: bool, record: bool = True) -> StandardPdhgOptions:
    s, beta, tol, limit = G[f"{name}/params"]
    return StandardPdhgOptions(step_size=float(s), restart_decay=float(beta), convergence_tol=float(tol),
                               iteration_limit=int(limit), record_iterates=record, parity=parity)


@pytest.mark.parametrize("name", NAMES)
def test_parity_mode_bitwise(name):
    lp = instance(name)
    assert spectral_norm(lp.constraint_matrix, 1e-12, 100000, parity=True) == G[f"{name}/norm"][0]
    for t in range(len(G[f"{name}/kkt_pts"])):
        x, y = G[f"{name}/pts_x"][t], G[f"{name}/pts_y"][t]
        assert kkt_error_standard(lp, x, y, parity=True) == G[f"{name}/kkt_pts"][t]
        s = float(G[f"{name}/params"][0])
        assert p_s_norm_squared(lp, s, x, y, parity=True) == G[f"{name}/ps_pts"][t]
    tr = restarted_pdhg_standard(lp, options(name, True), max_recorded=len(G[f"{name}/iter_x"]))
    cnt = G[f"{name}/counters"]
    assert (len(tr.epochs), tr.total_iterations, tr.converged, tr.numerical_failure) == \
        (cnt[0], cnt[1], bool(cnt[2]), bool(cnt[3]))
    assert np.array_equal([e.start_kkt for e in tr.epochs], G[f"{name}/kkt"])
    assert np.array_equal([e.length for e in tr.epochs], G[f"{name}/lens"])
    assert np.array_equal(tr.epochs[-1].start.primal, G[f"{name}/x_last"])
    assert np.array_equal(tr.epochs[-1].start.dual, G[f"{name}/y_last"])
    its = [z for e in tr.epochs for z in e.iterates]
    assert np.array_equal(np.array([z.primal for z in its]), G[f"{name}/iter_x"])
    assert np.array_equal(np.array([z.dual for z in its]), G[f"{name}/iter_y"])


@pytest.mark.parametrize("name", NAMES)
def test_fast_mode_matches_reference_and_theorem(name):
    lp = instance(name)
    nrm = spectral_norm(lp.constraint_matrix, 1e-12, 100000)
    assert nrm == pytest.approx(G[f"{name}/norm"][0], rel=1e-11)
    for t in range(len(G[f"{name}/kkt_pts"])):
        x, y = G[f"{name}/pts_x"][t], G[f"{name}/pts_y"][t]
        assert kkt_error_standard(lp, x, y) == pytest.approx(G[f"{name}/kkt_pts"][t], rel=1e-13)
        s = float(G[f"{name}/params"][0])
        assert p_s_norm_squared(lp, s, x, y) == pytest.approx(G[f"{name}/ps_pts"][t], rel=1e-12, abs=1e-12)
    opt = options(name, False)
    tr = restarted_pdhg_standard(lp, opt, max_recorded=len(G[f"{name}/iter_x"]))
    cnt = G[f"{name}/counters"]
    assert tr.converged == bool(cnt[2]) and not tr.numerical_failure
    # the first recorded iterates follow the reference's to fp64 round-off
    its = [z for e in tr.epochs for z in e.iterates]
    zx = np.array([np.concatenate([z.primal, z.dual]) for z in its][:100])
    zr = np.concatenate([G[f"{name}/iter_x"], G[f"{name}/iter_y"]], axis=1)[:100]
    assert np.max(np.linalg.norm(zx - zr, axis=1) / np.maximum(np.linalg.norm(zr, axis=1), 1e-300)) <= 1e-10
    # Theorem (iii): KKT(z^{n,0}) <= beta^n KKT(z^{0,0})
    kkt = np.array([e.start_kkt for e in tr.epochs])
    bound = kkt[0] * opt.restart_decay ** np.arange(len(kkt))
    assert np.all(kkt <= bound * (1.0 + 1e-10))
    if tr.converged:
        assert kkt[-1] <= opt.convergence_tol and len(kkt) >= 9  # criterion 5: >= 8 decay steps
        assert abs(tr.total_iterations - cnt[1]) <= 0.05 * cnt[1] + 64


@pytest.mark.parametrize("name", ["f1", "f4", "r30x60"])
def test_p_s_distance_to_optimum_nonincreasing_within_epochs(name):
    """acceptance_main.cpp:296-319, with z* = the converged point of a long run."""
    lp = instance(name)
    opt = options(name, False)
    ref = restarted_pdhg_standard(lp, StandardPdhgOptions(step_size=opt.step_size, convergence_tol=1e-13,
                                                          iteration_limit=2_000_000), max_recorded=0)
    zs = ref.epochs[-1].start
    tr = restarted_pdhg_standard(lp, opt, max_recorded=4000)
    s = opt.step_size
    dist = lambda z: np.sqrt(max(p_s_norm_squared(lp, s, z.primal - zs.primal, z.dual - zs.dual), 0.0))  # noqa: E731
    checked = 0
    for e in tr.epochs:
        seq = ([e.start] if e.start is not None else []) + e.iterates
        for a, b in zip(seq, seq[1:]):
            assert dist(b) <= dist(a) + 1e-9
            checked += 1
    assert checked > 0


@pytest.mark.parametrize("parity", [True, False])
def test_already_optimal_start_restart_chain(parity):
    """test_standard_form.cpp:112-127."""
    lp = instance("f0")
    tr = restarted_pdhg_standard(lp, StandardPdhgOptions(step_size=0.4, convergence_tol=-1.0, iteration_limit=10,
                                                         parity=parity),
                                 start=PrimalDualPoint(np.ones(1), np.ones(1)))
    cnt = G["chain/counters"]
    assert (len(tr.epochs), tr.total_iterations) == (cnt[0], cnt[1]) == (len(tr.epochs), 10)
    assert all(e.start_kkt == 0.0 and e.length <= 1 for e in tr.epochs)
    assert np.array_equal([e.length for e in tr.epochs], G["chain/lens"])


def test_invalid_options_rejected_through_the_c_abi():
    import ctypes as C

    from paper_2311_12180_b200.standard_form import _Csr, _lib

    lp = instance("f1")
    a = _Csr(lp.constraint_matrix)
    lib = _lib()
    o = abi.PdlpStandardOptions()
    lib.pdlp_standard_default_options(C.byref(o))
    cnt = np.zeros(4, np.int64)
    b, c = np.ascontiguousarray(lp.rhs), np.ascontiguousarray(lp.objective)
    for step, beta, msg in ((0.0, 0.5, b"step_size must be positive"), (0.1, 1.0, b"restart_decay must lie")):
        o.step_size, o.restart_decay = step, beta
        rc = lib.pdlp_standard_pdhg(C.byref(a.c), abi.dptr(b), abi.dptr(c), C.byref(o), None, None, None, None, 0,
                                    abi.i64ptr(cnt), None, None, None, None, 0)
        assert rc == abi.PDLP_EINVAL
        lib.pdlp_last_error.restype = C.c_char_p
        assert lib.pdlp_last_error().startswith(msg)
    with pytest.raises(ValueError, match="step_size must be positive"):
        StandardPdhgOptions(step_size=-1.0).validate()


def test_spectral_norm_of_empty_and_identity():
    ident = CsrMatrix(4, 4, np.arange(5, dtype=np.int64), np.arange(4, dtype=np.int64), np.ones(4))
    assert spectral_norm(ident) == pytest.approx(1.0, abs=1e-9)
    diag = CsrMatrix(3, 3, np.arange(4, dtype=np.int64), np.arange(3, dtype=np.int64), np.array([1.0, -3.0, 2.0]))
    assert spectral_norm(diag, 1e-14, 100000) == pytest.approx(3.0, abs=1e-8)
    empty = CsrMatrix(2, 3, np.zeros(3, np.int64), np.zeros(0, np.int64), np.zeros(0))
    assert spectral_norm(empty) == 0.0


@pytest.mark.parametrize("parity", [True, False])
def test_numerical_failure_and_limit_edges(parity):
    """A step far beyond 1/||A|| diverges to a non-finite iterate: the loop
    ends with numerical_failure and without counting the failed step
    (standard_form.hpp:177-180); iteration_limit 0 opens the first epoch only."""
    lp = instance("f4")
    tr = restarted_pdhg_standard(lp, StandardPdhgOptions(step_size=1e150, convergence_tol=1e-12,
                                                         iteration_limit=100000, parity=parity))
    assert tr.numerical_failure and not tr.converged
    cnt = G["fail/counters"]  # the reference's run of the same case
    assert (len(tr.epochs), tr.total_iterations, tr.converged, tr.numerical_failure) == \
        (cnt[0], cnt[1], bool(cnt[2]), bool(cnt[3]))
    assert np.array_equal([e.length for e in tr.epochs], G["fail/lens"])
    tr0 = restarted_pdhg_standard(lp, StandardPdhgOptions(step_size=0.1, iteration_limit=0, parity=parity))
    assert (tr0.total_iterations, len(tr0.epochs), tr0.converged) == (0, 1, False)
    assert tr0.epochs[0].start_kkt == pytest.approx(G["f4/kkt"][0], rel=0 if parity else 1e-14)
