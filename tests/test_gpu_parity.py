"""GPU parity tests: the CUDA product path (libpdlp_b200.so through the C-ABI)
against the CPU oracle (pinned bitwise to the reference) and the reference's
golden vectors.

Bars (BASELINE.json north_star): integer work bit-exact; parity mode bitwise
equal to the reference; fast mode's first 100 iterates within 1e-10 relative;
final status and objective agreeing within the solve tolerance.
"""
from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as O
from paper_2311_12180_b200 import Mode, Solver, SolverParams, SolveStatus, abi, generators, solve
from paper_2311_12180_b200.lp import CsrMatrix, GeneralFormLp
from tests.helpers import load_golden_lp, lp_hash, ref_c1, ref_suite, rel_err, sha, stacked_k, suite_names

pytestmark = pytest.mark.gpu

PARITY = SolverParams(mode=Mode.PARITY)


def skewed_lp(seed: int = 7) -> GeneralFormLp:
    """Rows from length 0 to 20000 (STREAM, WARP and split CHUNK tiles)."""
    rng = np.random.default_rng(seed)
    n = 30000
    lens = [0, 1, 2, 5, 31, 32, 33, 64, 200, 512, 513, 1000, 4095, 4096, 4097, 9000, 20000, 3, 7]
    lens += list(rng.integers(1, 40, size=300))
    rows, cols, vals = [], [], []
    for r, L in enumerate(lens):
        c = rng.choice(n, size=int(L), replace=False)
        rows += [r] * int(L)
        cols += list(c)
        vals += list(rng.uniform(-3, 3, size=int(L)))
    m = len(lens)
    m1 = m // 2
    K = CsrMatrix.from_triplets(m, n, rows, cols, vals)
    G = CsrMatrix(m1, n, K.row_offsets[: m1 + 1], K.col_indices[: K.row_offsets[m1]], K.values[: K.row_offsets[m1]])
    A = CsrMatrix(m - m1, n, K.row_offsets[m1:] - K.row_offsets[m1], K.col_indices[K.row_offsets[m1]:],
                  K.values[K.row_offsets[m1]:])
    return GeneralFormLp(G, A, rng.uniform(-1, 1, n), rng.uniform(-1, 1, m1), rng.uniform(-1, 1, m - m1),
                         np.zeros(n), np.full(n, 10.0))


# ---------------------------------------------------------------------------
# kernels: SpMV, transpose, scaling
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("mode", [Mode.FAST, Mode.PARITY])
@pytest.mark.parametrize("which", ["C1", "transport", "skewed"])
def test_spmv_against_oracle(mode, which):
    lp = {"C1": lambda: generators.config("C1"), "transport": lambda: generators.transport_lp(40, 70, seed=3),
          "skewed": skewed_lp}[which]()
    K = stacked_k(lp)
    rng = np.random.default_rng(1)
    x, y = rng.standard_normal(lp.num_variables), rng.standard_normal(lp.num_constraints)
    with Solver(lp, SolverParams(mode=mode)) as s:
        kx = s.spmv(abi.OP_K_ORIGINAL, x)
        kty = s.spmv(abi.OP_KT_ORIGINAL, y)
        d1, d2 = s.scaling()
        kxs = s.spmv(abi.OP_K_SCALED, x)
    ref_kx = O.spmv(K, x)
    ref_kty = O.spmv_transpose(K, y)
    lens = np.diff(K.row_offsets)
    stream_rows = lens <= 32
    if mode == Mode.PARITY:
        assert np.array_equal(kx, ref_kx)
        assert np.array_equal(kty, ref_kty)  # gather over stored K^T == scatter
    else:
        # STREAM rows are summed in index order: bitwise; longer rows: tree order
        assert np.array_equal(kx[stream_rows], ref_kx[stream_rows])
        assert rel_err(kx, ref_kx) <= 1e-13
        assert rel_err(kty, ref_kty) <= 1e-13
    # scaled operator: values v * (d1 * d2)
    Ks = CsrMatrix(K.num_rows, K.num_cols, K.row_offsets, K.col_indices,
                   K.values * (np.repeat(d1, lens) * d2[K.col_indices]))
    assert rel_err(kxs, O.spmv(Ks, x)) <= 1e-13


def test_transpose_bitwise_c1():
    lp = generators.config("C1")
    g = ref_c1()
    assert lp_hash(lp) == g["lp_sha256"]
    K = stacked_k(lp)
    kt = O.transpose(K)
    assert sha(kt.row_offsets, kt.col_indices, kt.values) == g["transpose_sha256"]
    # the device K^T (via the original K^T operator applied to unit vectors is too
    # slow); check K^T y against the scatter for y with distinct powers of two
    rng = np.random.default_rng(5)
    y = rng.standard_normal(lp.num_constraints)
    with Solver(lp, PARITY) as s:
        assert np.array_equal(s.spmv(abi.OP_KT_ORIGINAL, y), O.spmv_transpose(K, y))


@pytest.mark.parametrize("name", ["C1", "rand05", "blend", "transport23", "skewed"])
def test_scaling_bitwise(name):
    lp = generators.config("C1") if name == "C1" else skewed_lp() if name == "skewed" else load_golden_lp(name)
    for mode in (Mode.FAST, Mode.PARITY):
        with Solver(lp, SolverParams(mode=mode)) as s:
            d1, d2 = s.scaling()
        r1, r2 = O.scaling(lp)
        assert np.array_equal(d1, r1) and np.array_equal(d2, r2)
    if name == "C1":
        assert sha(d1, d2) == ref_c1()["scaling_sha256"]


def test_scaling_bitwise_on_eight_decade_matrices():
    """acceptance criterion 6's matrices (acceptance_main.cpp:340-421): entries
    +-10^U(-4, 4), 30% dense, every row and column used. The device's Ruiz(10) +
    Pock-Chambolle scaling equals the reference's bit for bit (so it also lands
    where the reference does: criterion 6 fails by design in the reference,
    10 Ruiz passes leave ~1.8e-2 of 8 decades)."""
    rng = np.random.default_rng(8080)
    for trial in range(12):
        rows, cols = int(rng.integers(5, 35)), int(rng.integers(5, 35))
        dense = rng.uniform(0, 1, (rows, cols)) < 0.3
        for r in np.flatnonzero(~dense.any(axis=1)):
            dense[r, rng.integers(cols)] = True
        for c in np.flatnonzero(~dense.any(axis=0)):
            dense[rng.integers(rows), c] = True
        vals = np.where(rng.uniform(0, 1, (rows, cols)) < 0.5, -1.0, 1.0) * 10.0 ** rng.uniform(-4, 4, (rows, cols))
        rr, cc = np.nonzero(dense)
        K = CsrMatrix.from_triplets(rows, cols, rr, cc, vals[rr, cc])
        m1 = rows // 2
        G = CsrMatrix(m1, cols, K.row_offsets[: m1 + 1], K.col_indices[: K.row_offsets[m1]],
                      K.values[: K.row_offsets[m1]])
        A = CsrMatrix(rows - m1, cols, K.row_offsets[m1:] - K.row_offsets[m1], K.col_indices[K.row_offsets[m1]:],
                      K.values[K.row_offsets[m1]:])
        lp = GeneralFormLp(G, A, rng.uniform(-1, 1, cols), rng.uniform(-1, 1, m1), rng.uniform(-1, 1, rows - m1),
                           np.zeros(cols), np.full(cols, np.inf))
        with Solver(lp, SolverParams()) as s:
            d1, d2 = s.scaling()
        r1, r2 = O.scaling(lp)
        assert np.array_equal(d1, r1) and np.array_equal(d2, r2), trial


# ---------------------------------------------------------------------------
# parity mode: the whole loop bitwise equal to the reference
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("name", suite_names())
def test_parity_mode_suite_bitwise(name):
    lp = load_golden_lp(name)
    ref = ref_suite()[name]
    assert lp_hash(lp) == ref["lp_sha256"]
    limit = 10000 if name.startswith("infeasible") else 1_000_000
    p = SolverParams(eps_optimal=1e-8, time_limit_seconds=60.0, iteration_limit=limit,
                     record_step_log=True, mode=Mode.PARITY)
    r = solve(lp, p)
    assert str(r.status) == ref["status"]
    assert r.iterations == ref["iterations"]
    assert r.restarts == ref["restarts"]
    assert sha(r.point.primal, r.point.dual) == ref["point_sha256"]
    assert sha(r.reduced.lambda_) == ref["lambda_sha256"]
    assert sha(r.step_log) == ref["step_log_sha256"]
    got = [[int(e["total_iterations"]), int(e["epoch_length"]), int(e["criterion"]),
            int(e["candidate_is_average"]), float(e["omega_after"])] for e in r.restart_log]
    assert got == ref["restart_log"]
    assert r.info["primal_objective"] == ref["primal_objective"]


@pytest.mark.parametrize("name", ["twovar", "degen", "prodmix", "rand01", "rand04"])
def test_parity_mode_eager_restarts(name):
    lp = load_golden_lp(name)
    ref = ref_suite()[name + "_eager"]
    p = SolverParams(eps_optimal=1e-8, time_limit_seconds=60.0, iteration_limit=1_000_000,
                     evaluation_frequency=1, record_step_log=True, mode=Mode.PARITY)
    r = solve(lp, p)
    assert (str(r.status), r.iterations, r.restarts) == (ref["status"], ref["iterations"], ref["restarts"])
    assert sha(r.point.primal, r.point.dual) == ref["point_sha256"]


def test_parity_mode_c1_first_100_iterates_bitwise():
    lp = generators.config("C1")
    g = ref_c1()
    with Solver(lp, PARITY) as s:
        s.iterate_begin()
        for k, (total, inner, outer, h, eta, omega) in enumerate(g["iterates"], start=1):
            s.iterate_run(1)
            it = s.iterate()
            assert (it["total"], it["inner"], it["outer"]) == (total, inner, outer)
            assert sha(it["x"], it["y"], it["kx"], it["kty"]) == h, f"iterate {k}"
            assert it["eta"] == eta and it["omega"] == omega


def test_parity_mode_c1_solve_bitwise():
    lp = generators.config("C1")
    g = ref_c1()["solve_1e-4"]
    r = solve(lp, PARITY)
    assert (str(r.status), r.iterations, r.restarts) == (g["status"], g["iterations"], g["restarts"])
    assert sha(r.point.primal, r.point.dual) == g["point_sha256"]


# ---------------------------------------------------------------------------
# fast mode: tolerance parity
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("which", ["C1", "transport", "skewed"])
def test_fast_mode_first_100_iterates(which):
    """First 100 iterates within 1e-10 relative (BASELINE.json north_star)."""
    lp = {"C1": lambda: generators.config("C1"), "transport": lambda: generators.transport_lp(60, 80, seed=11),
          "skewed": skewed_lp}[which]()
    ref = O.Session(lp, SolverParams(), "oracle")
    traj = []
    with Solver(lp, SolverParams()) as s:
        s.iterate_begin()
        for k in range(100):
            s.iterate_run(1)
            ref.run(1)
            a, b = s.iterate(), ref.iterate()
            assert (a["total"], a["inner"], a["outer"]) == (b["total"], b["inner"], b["outer"])
            za, zb = np.concatenate([a["x"], a["y"]]), np.concatenate([b["x"], b["y"]])
            # relative error of the iterate z = (x, y) in the 2-norm
            e = float(np.linalg.norm(za - zb) / max(np.linalg.norm(zb), 1e-300))
            traj.append((k + 1, e, rel_err(za, zb)))
    ref.close()
    print("iterate rel err (k, 2-norm, max-norm):", traj[::10], traj[-1])
    worst = max(e for _, e, _ in traj)
    assert worst <= 1e-10, f"worst relative iterate error {worst}"


def reorder_floor(lp, iters: int) -> tuple[float, float]:
    """The oracle against itself with pairwise step-size sums (sum order 1):
    how far a reordering alone moves the reference's first iterates."""
    a = O.Session(lp, SolverParams(), "oracle")
    O.set_sum_order(1)
    try:
        b = O.Session(lp, SolverParams(), "oracle")
        w2 = wi = 0.0
        for _ in range(iters):
            O.set_sum_order(0)
            a.run(1)
            O.set_sum_order(1)
            b.run(1)
            ia, ib = a.iterate(), b.iterate()
            za, zb = np.concatenate([ia["x"], ia["y"]]), np.concatenate([ib["x"], ib["y"]])
            w2 = max(w2, float(np.linalg.norm(zb - za) / max(np.linalg.norm(za), 1e-300)))
            wi = max(wi, rel_err(zb, za))
        b.close()
    finally:
        O.set_sum_order(0)
    a.close()
    return w2, wi


@pytest.mark.parametrize("which", ["staircase", "multicommodity"])
def test_fast_mode_drift_small_tile_band(which):
    """Structured operators in the 64k-256k nnz band, where the iteration
    tiles are 1024-nnz STREAM tiles (solver.cu build_plan): the first 100
    iterates within 1e-10, or within 4x the reference's own reordering drift
    on the same instance where that floor is higher."""
    lp = {"staircase": lambda: generators.staircase_lp(3, 5000, 1250, 1250, seed=12),
          "multicommodity": lambda: generators.multicommodity_lp(600, 4000, 6, seed=13)}[which]()
    assert (1 << 16) <= lp.nnz < (1 << 18), lp.nnz
    ref = O.Session(lp, SolverParams(), "oracle")
    w2 = wi = 0.0
    with Solver(lp, SolverParams()) as s:
        s.iterate_begin()
        for _ in range(100):
            s.iterate_run(1)
            ref.run(1)
            a, b = s.iterate(), ref.iterate()
            assert (a["total"], a["inner"]) == (b["total"], b["inner"])
            za, zb = np.concatenate([a["x"], a["y"]]), np.concatenate([b["x"], b["y"]])
            w2 = max(w2, float(np.linalg.norm(za - zb) / max(np.linalg.norm(zb), 1e-300)))
            wi = max(wi, rel_err(za, zb))
    ref.close()
    f2, fi = reorder_floor(lp, 100)
    print(f"{which} nnz {lp.nnz}: fast {w2:.3e} / {wi:.3e}, reorder floor {f2:.3e} / {fi:.3e}")
    assert w2 <= max(1e-10, 4.0 * f2) and wi <= max(1e-10, 4.0 * fi), (w2, wi, f2, fi)


@pytest.mark.parametrize("which", ["C1", "transport", "rand09", "blend"])
def test_fast_mode_solve_status_and_objective(which):
    lp = {"C1": lambda: generators.config("C1"), "transport": lambda: generators.transport_lp(60, 80, seed=11),
          "rand09": lambda: load_golden_lp("rand09"), "blend": lambda: load_golden_lp("blend")}[which]()
    eps = 1e-4 if which in ("C1", "transport") else 1e-8
    p = SolverParams(eps_optimal=eps, iteration_limit=1_000_000, time_limit_seconds=120.0)
    r = solve(lp, p)
    ref = O.solve(lp, p)
    assert r.status == ref.status == SolveStatus.OPTIMAL
    obj, robj = r.info["primal_objective"], ref.info["primal_objective"]
    assert abs(obj - robj) <= 2 * eps * (1.0 + abs(robj))
    # the reference's own criteria hold at the GPU's point (criterion 2 style)
    chk = O.check_termination(lp, r.point.primal, r.point.dual, eps)
    assert chk["terminated"]


def test_fast_mode_deterministic():
    lp = generators.transport_lp(60, 80, seed=11)
    p = SolverParams(record_step_log=True)
    a, b = solve(lp, p), solve(lp, p)
    assert a.iterations == b.iterations and a.restarts == b.restarts
    assert np.array_equal(a.point.primal, b.point.primal) and np.array_equal(a.point.dual, b.point.dual)
    assert np.array_equal(a.step_log, b.step_log)


def test_split_rows_deterministic_across_runs():
    """Split rows (CHUNK tiles) are finished by whichever slice CTA arrives
    last; their reduction terms must still land in a fixed partial slot, or the
    step sizes drift in the last bits from run to run (seen as ~20% of runs
    differing before the fix)."""
    lp = skewed_lp()
    hashes, solves = set(), set()
    for engine in (abi.ENGINE_GRAPH, abi.ENGINE_STREAM):
        for _ in range(8):
            with Solver(lp, SolverParams(eps_optimal=1e-6, iteration_limit=2, engine=engine)) as s:
                s.iterate_begin()
                s.iterate_run(2)
                it = s.iterate()
                hashes.add(sha(np.concatenate([it["x"], it["y"], it["kx"]])))
        for _ in range(3):
            r = solve(lp, SolverParams(eps_optimal=1e-6, engine=engine))
            solves.add((r.iterations, sha(r.point.primal), sha(r.point.dual)))
    assert len(hashes) == 1 and len(solves) == 1, (hashes, solves)


def test_two_suite_runs_bitwise_identical():
    """acceptance criterion 9 (acceptance_main.cpp:522-544) in fast mode: every
    suite instance solved twice gives the same status, iteration count, point
    and objective bit for bit."""
    p = SolverParams(eps_optimal=1e-8, iteration_limit=200000)
    for name in suite_names():
        lp = load_golden_lp(name)
        a, b = solve(lp, p), solve(lp, p)
        assert (a.status, a.iterations) == (b.status, b.iterations), name
        assert sha(a.point.primal, a.point.dual) == sha(b.point.primal, b.point.dual), name
        assert a.info["primal_objective"] == b.info["primal_objective"] or \
            (np.isnan(a.info["primal_objective"]) and np.isnan(b.info["primal_objective"])), name


@pytest.mark.parametrize("which", ["C1", "transport", "skewed", "staircase", "infeasible_primal", "rand07",
                                   "C1_limit"])
def test_chained_windows_bitwise_equal_to_host_decided(which, monkeypatch):
    """Windows chained on the device (the evaluation's no-restart decision
    taken by chain_decide_kernel) give the same solve as the host deciding
    after every window: status, iteration and restart counts, restart log,
    point and objective, bit for bit."""
    lp = {"C1": lambda: generators.config("C1"), "C1_limit": lambda: generators.config("C1"),
          "transport": lambda: generators.transport_lp(60, 80, seed=11), "skewed": skewed_lp,
          "staircase": lambda: generators.staircase_lp(3, 2000, 500, 500, seed=8)}.get(
              which, lambda: load_golden_lp(which))()
    p = SolverParams(eps_optimal=1e-8, iteration_limit=1000 if which == "C1_limit" else 400000)
    a = solve(lp, p)
    monkeypatch.setenv("PDLP_NO_CHAIN", "1")
    b = solve(lp, p)
    assert (a.status, a.iterations, a.restarts) == (b.status, b.iterations, b.restarts), which
    assert np.array_equal(a.restart_log, b.restart_log)
    assert sha(a.point.primal, a.point.dual, a.reduced.lambda_) == sha(b.point.primal, b.point.dual, b.reduced.lambda_)
    assert a.info["primal_objective"] == b.info["primal_objective"] or np.isnan(a.info["primal_objective"])
    assert a.info["evaluations"] == b.info["evaluations"]


def test_graph_and_stream_engines_bitwise():
    """Same per-trial kernels, replayed by a CUDA graph or launched one by one."""
    lp = generators.config("C1")
    a = solve(lp, SolverParams(engine=abi.ENGINE_GRAPH))
    b = solve(lp, SolverParams(engine=abi.ENGINE_STREAM))
    assert a.iterations == b.iterations
    assert np.array_equal(a.point.primal, b.point.primal)




# ---------------------------------------------------------------------------
# behaviour mirrored from the reference's unit tests (test_solver.cpp)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("mode", [Mode.FAST, Mode.PARITY])
def test_infeasibility_certificates(mode):
    for name, status in (("infeasible_primal", SolveStatus.PRIMAL_INFEASIBLE),
                         ("infeasible_dual", SolveStatus.DUAL_INFEASIBLE)):
        lp = load_golden_lp(name)
        r = solve(lp, SolverParams(eps_optimal=1e-8, iteration_limit=10000, mode=mode))
        assert r.status == status and r.certificate is not None
        if status == SolveStatus.PRIMAL_INFEASIBLE:  # exact Farkas recheck (criterion 7)
            yv = r.certificate.dual_ray
            yn = np.linalg.norm(yv)
            assert yn > 0 and (yv[: lp.num_inequalities] >= 0).all()
            K = stacked_k(lp)
            kty = O.spmv_transpose(K, yv) + r.certificate.dual_ray_reduced_costs.lambda_
            assert np.linalg.norm(kty) <= 1e-8 * yn
        else:
            xv = r.certificate.primal_ray
            assert np.linalg.norm(xv) > 0 and lp.objective @ xv < -1e-8 * np.linalg.norm(xv)


def test_limits():
    lp = generators.small_random_lp(4, 2, 1, seed=3)
    r = solve(lp, SolverParams(eps_optimal=1e-14, iteration_limit=10))
    assert r.status == SolveStatus.ITERATION_LIMIT and r.iterations == 10
    r = solve(lp, SolverParams(eps_optimal=1e-14, time_limit_seconds=0.0))
    assert r.status == SolveStatus.TIME_LIMIT


def test_step_log_contract():
    """test_solver.cpp:483-505: eta' follows the min formula bitwise."""
    import math

    lp = load_golden_lp("rand03")
    r = solve(lp, SolverParams(eps_optimal=1e-8, record_step_log=True))
    assert r.status == SolveStatus.OPTIMAL and len(r.step_log) == r.iterations
    for e in r.step_log:
        if e["interaction"] != 0.0:
            assert e["eta_bar"] == e["movement_sq"] / (2.0 * abs(e["interaction"]))
        kp1 = float(e["step_counter"]) + 1.0
        exp = min((1.0 - math.pow(kp1, -0.3)) * e["eta_bar"], (1.0 + math.pow(kp1, -0.6)) * e["eta_accepted"])
        assert e["eta_next"] == exp


def test_zero_matrix_and_empty_rows():
    # min -x s.t. 0 >= -1 (no stored entries), x in [0, 10]: test_solver.cpp:64-75
    G = CsrMatrix(1, 1, np.array([0, 0]), np.zeros(0, np.int64), np.zeros(0))
    A = CsrMatrix.zero(0, 1)
    lp = GeneralFormLp(G, A, np.array([-1.0]), np.array([-1.0]), np.zeros(0), np.zeros(1), np.array([10.0]))
    r = solve(lp, SolverParams(eps_optimal=1e-8))
    ref = O.solve(lp, SolverParams(eps_optimal=1e-8))
    assert r.status == ref.status and r.iterations == ref.iterations


def test_invalid_input_raises_value_error():
    lp = generators.small_random_lp(3, 1, 1, seed=2)
    with pytest.raises(ValueError, match="tolerances must be positive"):
        Solver(lp, SolverParams(eps_optimal=0.0))
    bad = generators.small_random_lp(3, 1, 1, seed=2)
    bad.lower[1] = 5.0
    bad.upper[1] = 1.0
    with pytest.raises(ValueError, match="empty bound interval on variable 1"):
        Solver(bad, SolverParams())


# ---------------------------------------------------------------------------
# GPU CSR construction (sparse_matrix.hpp:57-108)
# ---------------------------------------------------------------------------

def test_gpu_from_triplets_matches_oracle():
    from paper_2311_12180_b200.api import csr_from_triplets

    rng = np.random.default_rng(5)
    for trial in range(30):
        rows, cols = int(rng.integers(1, 300)), int(rng.integers(1, 300))
        t = int(rng.integers(0, 3000))
        r, c = rng.integers(0, rows, t), rng.integers(0, cols, t)
        v = rng.uniform(-5, 5, t)
        v[rng.uniform(size=t) < 0.05] = 0.0
        if t > 4:  # exact cancellation of a duplicated pair: the entry is dropped
            r[-1], c[-1], v[-1] = r[0], c[0], -v[0]
        g = csr_from_triplets(rows, cols, r, c, v)
        o = O.from_triplets(rows, cols, r, c, v)
        assert np.array_equal(g.row_offsets, o.row_offsets)  # integer work: bit-exact
        assert np.array_equal(g.col_indices, o.col_indices)
        _, mult = np.unique(r * cols + c, return_counts=True)
        if mult.max(initial=0) <= 2:
            assert np.array_equal(g.values, o.values)
        else:
            assert np.allclose(g.values, o.values, rtol=1e-13, atol=1e-13)
    with pytest.raises(ValueError, match="triplet 1 at \\(2, 0\\) is outside a 2x2 matrix"):
        csr_from_triplets(2, 2, [0, 2, 5], [0, 0, 0], [1.0, 1.0, 1.0])
    e = csr_from_triplets(3, 4, [], [], [])
    assert list(e.row_offsets) == [0, 0, 0, 0] and e.nnz == 0


def test_gpu_from_triplets_large_matches_host_csr():
    from paper_2311_12180_b200.api import csr_from_triplets

    lp = generators.config("C1")
    K = stacked_k(lp)
    rows = np.repeat(np.arange(K.num_rows), np.diff(K.row_offsets))
    perm = np.random.default_rng(3).permutation(K.nnz)
    g = csr_from_triplets(K.num_rows, K.num_cols, rows[perm], K.col_indices[perm], K.values[perm])
    assert np.array_equal(g.row_offsets, K.row_offsets) and np.array_equal(g.col_indices, K.col_indices)
    assert np.array_equal(g.values, K.values)


# ---------------------------------------------------------------------------
# column panels (panels.cu): forced on small instances with narrow panels
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("width", ["700", "4096", "1000000000"])  # the last: one panel (C5's single-panel sweep)
def test_column_panel_spmv_bitwise_sequential(width, monkeypatch):
    """The panel sweep sums every row by one thread in column order, from 0.0:
    bitwise equal to the reference's sequential spmv (sparse_matrix.hpp:117-132)
    over K and to spmv_transpose (:142-158) over the stored K^T."""
    monkeypatch.setenv("PDLP_PANELS", "1")
    monkeypatch.setenv("PDLP_PANEL_WIDTH", width)
    lp = generators.config("C1")
    rng = np.random.default_rng(5)
    K = stacked_k(lp)
    lens = np.diff(K.row_offsets)
    with Solver(lp, SolverParams()) as s:
        d1, d2 = s.scaling()
        x = rng.uniform(-2, 2, lp.num_variables)
        y = rng.uniform(-2, 2, lp.num_constraints)
        kx = s.spmv(abi.OP_K_SCALED, x)
        kty = s.spmv(abi.OP_KT_SCALED, y)
    Ks = CsrMatrix(K.num_rows, K.num_cols, K.row_offsets, K.col_indices,
                   K.values * (np.repeat(d1, lens) * d2[K.col_indices]))  # v *= dr * dc, scaling.hpp:150-152
    assert np.array_equal(kx, O.spmv(Ks, x))
    assert np.array_equal(kty, O.spmv_transpose(Ks, y))


@pytest.mark.parametrize("which", ["C1", "transport", "skewed"])
def test_column_panels_match_oracle(which, monkeypatch):
    monkeypatch.setenv("PDLP_PANELS", "1")
    monkeypatch.setenv("PDLP_PANEL_WIDTH", "700")
    lp = {"C1": lambda: generators.config("C1"), "transport": lambda: generators.transport_lp(60, 80, seed=11),
          "skewed": skewed_lp}[which]()
    ref = O.Session(lp, SolverParams(), "oracle")
    with Solver(lp, SolverParams()) as s:
        s.iterate_begin()
        worst = 0.0
        for k in range(100):
            s.iterate_run(1)
            ref.run(1)
            a, b = s.iterate(), ref.iterate()
            assert (a["total"], a["inner"]) == (b["total"], b["inner"])
            za, zb = np.concatenate([a["x"], a["y"]]), np.concatenate([b["x"], b["y"]])
            worst = max(worst, float(np.linalg.norm(za - zb) / max(np.linalg.norm(zb), 1e-300)))
    ref.close()
    assert worst <= 1e-10, worst
    p = SolverParams(eps_optimal=1e-6, iteration_limit=200000)
    r, o = solve(lp, p), O.solve(lp, p)
    assert r.status == o.status
    if r.status == SolveStatus.OPTIMAL:
        assert abs(r.info["primal_objective"] - o.info["primal_objective"]) <= 1e-5 * (
            1.0 + abs(o.info["primal_objective"]))


# ---------------------------------------------------------------------------
# fast mode over the whole reference suite (acceptance criteria 1/2/7 style)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("name", [n for n in suite_names()])
def test_fast_mode_suite_status_objective_and_reference_check(name):
    """Every suite instance (acceptance_main.cpp:79-154, 425-504) in fast mode:
    same status as the reference; optimal points pass the reference's own
    termination check at 1e-8 (criterion 2) and match its objective."""
    lp = load_golden_lp(name)
    ref = ref_suite()[name]
    limit = 10000 if name.startswith("infeasible") else 1_000_000
    r = solve(lp, SolverParams(eps_optimal=1e-8, iteration_limit=limit, time_limit_seconds=60.0))
    assert str(r.status) == ref["status"]
    if r.status == SolveStatus.OPTIMAL:
        chk = O.check_termination(lp, r.point.primal, r.point.dual, 1e-8)
        assert chk["terminated"]
        assert abs(r.info["primal_objective"] - ref["primal_objective"]) <= 1e-6 * (
            1.0 + abs(ref["primal_objective"]))


@pytest.mark.parametrize("gen", ["multicommodity", "staircase"])
def test_fast_mode_structured_generators_match_oracle(gen):
    """The C3 / C5 generator shapes at small size: first 100 iterates within
    1e-10 relative of the oracle, same status and objective at 1e-6."""
    lp = {"multicommodity": lambda: generators.multicommodity_lp(300, 2000, 5, seed=4),
          "staircase": lambda: generators.staircase_lp(3, 2000, 500, 500, seed=8)}[gen]()
    ref = O.Session(lp, SolverParams(), "oracle")
    with Solver(lp, SolverParams()) as s:
        s.iterate_begin()
        worst = 0.0
        for k in range(100):
            s.iterate_run(1)
            ref.run(1)
            a, b = s.iterate(), ref.iterate()
            za, zb = np.concatenate([a["x"], a["y"]]), np.concatenate([b["x"], b["y"]])
            worst = max(worst, float(np.linalg.norm(za - zb) / max(np.linalg.norm(zb), 1e-300)))
    ref.close()
    assert worst <= 1e-10
    p = SolverParams(eps_optimal=1e-6, iteration_limit=200000)
    r, o = solve(lp, p), O.solve(lp, p)
    assert r.status == o.status == SolveStatus.OPTIMAL
    assert abs(r.info["primal_objective"] - o.info["primal_objective"]) <= 1e-5 * (1.0 + abs(o.info["primal_objective"]))
