"""CPU tests (no GPU): pin the oracle before trusting it.

The plain-C restatement (oracle/pdlp_oracle.c) must reproduce the REFERENCE
solver bitwise:
  * against the committed golden vectors generated from the reference
    (tests/golden/make_golden.py, oracle/_ref built from /root/reference);
  * against the reference harness itself when oracle/_ref is built (this
    container; the GPU box ships the prebuilt .so);
  * against the reference's own known-answer unit tests
    (proj/tests/test_sparse.cpp, test_solver.cpp) restated here.
"""
from __future__ import annotations

import json

import numpy as np
import pytest

from oracle import oracle as O
from paper_2311_12180_b200 import SolverParams, SolveStatus, generators
from paper_2311_12180_b200.lp import CsrMatrix, GeneralFormLp
from tests.helpers import GOLDEN, load_golden_lp, lp_hash, ref_c1, ref_suite, sha, stacked_k

SUITE = ref_suite()


def suite_params(key: str) -> SolverParams:
    """Exactly the parameters make_golden.py solved the reference with."""
    name = key.replace("_eager", "")
    limit = 10000 if name.startswith("infeasible") else 1_000_000
    return SolverParams(eps_optimal=1e-8, time_limit_seconds=60.0, iteration_limit=limit,
                        evaluation_frequency=1 if key.endswith("_eager") else 64, record_step_log=True)


@pytest.mark.parametrize("key", sorted(SUITE))
def test_oracle_suite_bitwise_vs_reference_golden(key):
    """Criteria 1/2/4/7 instances (acceptance_main.cpp:79-230,425-504): every
    status, count, point, step log and restart log equals the reference's."""
    e = SUITE[key]
    lp = load_golden_lp(key.replace("_eager", ""))
    assert lp_hash(lp) == e["lp_sha256"]
    r = O.solve(lp, suite_params(key), "oracle")
    assert str(r.status) == e["status"]
    assert r.iterations == e["iterations"]
    assert r.restarts == e["restarts"]
    assert sha(r.point.primal, r.point.dual) == e["point_sha256"]
    assert sha(r.reduced.lambda_) == e["lambda_sha256"]
    assert sha(r.step_log) == e["step_log_sha256"]
    got = [[int(v["total_iterations"]), int(v["epoch_length"]), int(v["criterion"]),
            int(v["candidate_is_average"]), float(v["omega_after"])] for v in r.restart_log]
    assert got == e["restart_log"]
    assert r.info["primal_objective"] == e["primal_objective"]


def test_oracle_suite_points_match_golden_arrays():
    pts = np.load(GOLDEN / "ref_suite_points.npz")
    for key in ("rand05", "transport23", "infeasible_primal", "twovar_eager"):
        r = O.solve(load_golden_lp(key.replace("_eager", "")), suite_params(key), "oracle")
        assert np.array_equal(r.point.primal, pts[key + "__x"])
        assert np.array_equal(r.point.dual, pts[key + "__y"])


def test_oracle_c1_first_100_iterates_bitwise():
    """The re-driven loop's first 100 iterates of C1 (SURVEY.md §8c mechanism 1)."""
    g = ref_c1()
    lp = generators.config("C1")
    assert lp_hash(lp) == g["lp_sha256"]
    s = O.Session(lp, SolverParams(), "oracle")
    for k, (total, inner, outer, h, eta, omega) in enumerate(g["iterates"], start=1):
        s.run(1)
        it = s.iterate()
        assert (it["total"], it["inner"], it["outer"]) == (total, inner, outer), k
        assert sha(it["x"], it["y"], it["kx"], it["kty"]) == h, f"iterate {k}"
        assert it["eta"] == eta and it["omega"] == omega
    z = np.load(GOLDEN / "ref_c1_iter100.npz")
    assert np.array_equal(it["x"], z["x"]) and np.array_equal(it["y"], z["y"])
    s.close()


def test_oracle_c1_scaling_transpose_and_solve_golden():
    g = ref_c1()
    lp = generators.config("C1")
    d1, d2 = O.scaling(lp, SolverParams(), "oracle")
    assert sha(d1, d2) == g["scaling_sha256"]
    kt = O.transpose(stacked_k(lp), "oracle")
    assert sha(kt.row_offsets, kt.col_indices, kt.values) == g["transpose_sha256"]
    r = O.solve(lp, SolverParams(), "oracle")
    s = g["solve_1e-4"]
    assert (str(r.status), r.iterations, r.restarts) == (s["status"], s["iterations"], s["restarts"])
    assert r.info["primal_objective"] == s["primal_objective"]
    assert sha(r.point.primal, r.point.dual) == s["point_sha256"]


# ---------------------------------------------------------------------------
# live comparison with the reference harness (oracle/_ref)
# ---------------------------------------------------------------------------

needs_ref = pytest.mark.skipif(not O.available("ref"), reason="oracle/_ref not built (needs /root/reference)")


@needs_ref
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_oracle_equals_reference_on_random_lps(seed):
    lp = generators.small_random_lp(12 + seed, 5, 4, seed=seed)
    p = SolverParams(eps_optimal=1e-8, record_step_log=True)
    a, b = O.solve(lp, p, "oracle"), O.solve(lp, p, "ref")
    assert (a.status, a.iterations, a.restarts) == (b.status, b.iterations, b.restarts)
    assert np.array_equal(a.point.primal, b.point.primal) and np.array_equal(a.point.dual, b.point.dual)
    assert np.array_equal(a.step_log, b.step_log)
    assert np.array_equal(a.restart_log, b.restart_log)


@needs_ref
def test_oracle_equals_reference_skewed_and_transport():
    for lp in (generators.transport_lp(30, 45, seed=9), generators.random_lp(300, 200, 900, 4, seed=5)):
        p = SolverParams(iteration_limit=700)
        a, b = O.solve(lp, p, "oracle"), O.solve(lp, p, "ref")
        assert a.iterations == b.iterations
        assert np.array_equal(a.point.primal, b.point.primal) and np.array_equal(a.point.dual, b.point.dual)
        d_o, d_r = O.scaling(lp, SolverParams(), "oracle"), O.scaling(lp, SolverParams(), "ref")
        assert np.array_equal(d_o[0], d_r[0]) and np.array_equal(d_o[1], d_r[1])


@needs_ref
def test_from_triplets_and_transpose_bitwise_vs_reference():
    rng = np.random.default_rng(11)
    for trial in range(20):
        rows, cols = int(rng.integers(1, 40)), int(rng.integers(1, 40))
        t = int(rng.integers(0, 200))
        r, c = rng.integers(0, rows, t), rng.integers(0, cols, t)
        v = rng.uniform(-5, 5, t)
        v[rng.uniform(size=t) < 0.05] = 0.0
        a = O.from_triplets(rows, cols, r, c, v, "oracle")
        b = O.from_triplets(rows, cols, r, c, v, "ref")
        assert np.array_equal(a.row_offsets, b.row_offsets)  # integer output: bit-exact
        assert np.array_equal(a.col_indices, b.col_indices)
        # a sum of >= 3 duplicates depends on std::sort's unstable order
        # (sparse_matrix.hpp:93-94): bitwise only for <= 2
        _, mult = np.unique(r * cols + c, return_counts=True)
        if mult.max(initial=0) <= 2:
            assert np.array_equal(a.values, b.values)
        else:
            assert np.allclose(a.values, b.values, rtol=1e-14, atol=1e-14)
        ta, tb = O.transpose(b, "oracle"), O.transpose(b, "ref")
        assert np.array_equal(ta.row_offsets, tb.row_offsets) and np.array_equal(ta.col_indices, tb.col_indices)
        assert np.array_equal(ta.values, tb.values)


# ---------------------------------------------------------------------------
# the reference's own known-answer tests (test_sparse.cpp:36-174)
# ---------------------------------------------------------------------------

def test_known_answer_from_triplets():
    m = O.from_triplets(2, 2, [0, 1], [0, 1], [1.0, 1.0])  # test_sparse.cpp:36-43
    assert list(m.row_offsets) == [0, 1, 2] and list(m.col_indices) == [0, 1] and list(m.values) == [1.0, 1.0]
    m = O.from_triplets(2, 2, [0, 0], [0, 0], [1.0, 2.0])  # :45-56 duplicates summed
    assert m.nnz == 1 and m.values[0] == 3.0
    m = O.from_triplets(2, 2, [0, 0, 1], [1, 1, 0], [2.5, -2.5, 1.0])  # exact zeros dropped
    assert m.nnz == 1 and list(m.col_indices) == [0]
    with pytest.raises(ValueError, match="triplet 1"):  # :58-62
        O.from_triplets(2, 2, [0, 2], [0, 0], [1.0, 1.0])


def test_known_answer_spmv():
    eye = CsrMatrix.identity(3)  # test_sparse.cpp:112-136
    x = np.array([1.0, -2.0, 0.5])
    assert np.array_equal(O.spmv(eye, x), x)
    m = CsrMatrix.from_triplets(2, 2, [0, 0, 1], [0, 1, 1], [1.0, 2.0, 3.0])
    assert list(O.spmv(m, [1.0, 1.0])) == [3.0, 3.0]
    assert list(O.spmv_transpose(m, [1.0, 1.0])) == [1.0, 5.0]
    assert np.array_equal(O.spmv(CsrMatrix.zero(4, 3), x), np.zeros(4))
    col = CsrMatrix.from_triplets(3, 1, [0, 1, 2], [0, 0, 0], [2.0, -1.0, 4.0])  # :138-144
    assert list(O.spmv_transpose(col, [1.0, 2.0, 3.0])) == [2.0 - 2.0 + 12.0]


def test_spmv_transpose_equals_gather_over_explicit_transpose_bitwise():
    """the scatter spmv_transpose equals a sequential gather
    over explicit_transpose(K) bit for bit — the basis of the stored-K^T design."""
    rng = np.random.default_rng(17)
    for trial in range(50):
        rows, cols = int(rng.integers(1, 50)), int(rng.integers(1, 50))
        d = np.where(rng.uniform(size=(rows, cols)) < 0.15, rng.uniform(-1, 1, (rows, cols)), 0.0)
        r, c = np.nonzero(d)
        m = CsrMatrix.from_triplets(rows, cols, r, c, d[r, c])
        y = rng.uniform(-1, 1, rows)
        assert np.array_equal(O.spmv_transpose(m, y), O.spmv(O.transpose(m), y))
        mtt = O.transpose(O.transpose(m))
        assert np.array_equal(mtt.row_offsets, m.row_offsets) and np.array_equal(mtt.values, m.values)


def test_spmv_linear():
    rng = np.random.default_rng(23)  # test_sparse.cpp:155-174
    for trial in range(30):
        rows, cols = int(rng.integers(1, 30)), int(rng.integers(1, 30))
        d = np.where(rng.uniform(size=(rows, cols)) < 0.3, rng.uniform(-1, 1, (rows, cols)), 0.0)
        r, c = np.nonzero(d)
        m = CsrMatrix.from_triplets(rows, cols, r, c, d[r, c])
        x, y = rng.uniform(-1, 1, cols), rng.uniform(-1, 1, cols)
        lhs = O.spmv(m, 1.75 * x - 0.5 * y)
        rhs = 1.75 * O.spmv(m, x) - 0.5 * O.spmv(m, y)
        assert np.all(np.abs(lhs - rhs) <= 1e-12 * np.maximum(1.0, np.abs(rhs)))


def test_known_answer_twovar_solve():
    """End-to-end known answer (test_solver.cpp:327-340 style): min x0 + x1,
    x0 + x1 >= 1, 0 <= x <= 10 has objective 1."""
    G = CsrMatrix.from_triplets(1, 2, [0, 0], [0, 1], [1.0, 1.0])
    lp = GeneralFormLp(G, CsrMatrix.zero(0, 2), [1.0, 1.0], [1.0], np.zeros(0), [0.0, 0.0], [10.0, 10.0])
    r = O.solve(lp, SolverParams(eps_optimal=1e-8))
    assert r.status == SolveStatus.OPTIMAL
    assert abs(r.info["primal_objective"] - 1.0) <= 1e-6


def test_golden_manifest_is_complete():
    names = {k.replace("_eager", "") for k in SUITE}
    assert len([n for n in names if n.startswith("rand") or n in
                ("assign22", "blend", "degen", "diet", "freevars", "knaprelax", "pathflow", "prodmix",
                 "transport23", "twovar")]) >= 20  # acceptance needs >= 20 suite instances
    assert json.loads((GOLDEN / "ref_c1.json").read_text())["nnz"] == 100000


def test_oracle_c2_first_100_iterates_match_reference_goldens():
    """The C restatement re-drives C2 (BASELINE configs[1], 2M nonzeros)
    exactly like the reference (tests/golden/make_golden_configs.py ran
    oracle/_ref): counters, step sizes, primal weight and the sampled iterate
    entries are bitwise equal over the first 100 iterations."""
    meta = json.loads((GOLDEN / "configs.json").read_text())["C2"]
    g = dict(np.load(GOLDEN / "configs_C2.npz"))
    lp = generators.config("C2")
    assert lp_hash(lp) == meta["instance_sha256"]
    s = O.Session(lp, SolverParams(), "oracle")
    for k in range(meta["iterates"]):
        s.run(1)
        it = s.iterate()
        for key in ("total", "inner", "trials", "eta", "eta_hat", "omega"):
            assert it[key] == g[key][k], (key, k)
        assert np.array_equal(it["x"][g["ix"]], g["x_s"][k]) and np.array_equal(it["y"][g["iy"]], g["y_s"][k]), k
        assert np.linalg.norm(it["x"]) == g["x_norm"][k] and np.linalg.norm(it["y"]) == g["y_norm"][k]
    s.close()


def test_c2_reorder_drift_matches_committed_floor():
    """configs.json `reorder_drift` (the floor of tests/test_gpu_configs.py's
    fast-mode bars) is reproducible: the C restatement re-run with pairwise
    step-size sums (oracle sum order 1) against its sequential self gives the
    committed C2 figures exactly, and a reordering alone already moves the
    reference's iterates."""
    import importlib.util

    spec = importlib.util.spec_from_file_location("mgc", GOLDEN / "make_golden_configs.py")
    mgc = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mgc)
    meta = json.loads((GOLDEN / "configs.json").read_text())["C2"]
    got = mgc.reorder_drift("C2", generators.config("C2"))
    assert got["rel2"] == meta["reorder_drift"]["rel2"] and got["relinf"] == meta["reorder_drift"]["relinf"]
    assert got["rel2"] > 0.0


def test_oracle_pdhg_raw_step_known_answers_and_reference():
    """pdhg_raw_step (solver.hpp:335-358): the reference's hand traces
    (test_solver.cpp:33-61) and bitwise equality with the reference compiled
    in place on a seeded LP."""
    from tests.test_gpu_raw_step import one_var_lp, origin_lp

    x, y = O.pdhg_raw_step(origin_lp(), np.zeros(2), np.zeros(1), 0.7, 0.3)
    assert x.tolist() == [0.0, 0.0] and y.tolist() == [0.0]
    x, y = O.pdhg_raw_step(one_var_lp(), np.zeros(1), np.zeros(1), 0.5, 0.5)
    assert x.tolist() == [0.0] and y.tolist() == [0.5]
    x, y = O.pdhg_raw_step(one_var_lp(), np.ones(1), np.ones(1), 0.4, 0.9)
    assert x.tolist() == [1.0] and y.tolist() == [1.0]
    if not O.available("ref"):
        pytest.skip("oracle/_ref not built")
    lp = generators.random_lp(60, 40, 150, 4, seed=9)
    rng = np.random.default_rng(9)
    xs, ys = rng.uniform(-1, 3, lp.num_variables), rng.uniform(-2, 2, lp.num_constraints)
    a, b = O.pdhg_raw_step(lp, xs, ys, 0.3, 0.7), O.pdhg_raw_step(lp, xs, ys, 0.3, 0.7, "ref")
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
