"""Regenerates tests/golden/ from the REFERENCE solver (oracle/_ref, built from
/root/reference by oracle/Makefile). Run in the build container only:

    make -C oracle ref && python tests/golden/make_golden.py

Outputs (committed; the GPU box has no /root/reference):
  suite/*.npz         the 21 suite instances + hand fixtures, parsed by the
                      reference's own MPS reader (mps_io.hpp:582)
  ref_suite.json      reference solve of each at eps 1e-8 (criteria 1/2 setup,
                      acceptance_main.cpp:60-75): status, iterations, restarts,
                      objective, sha256 of the returned point, restart log
  ref_suite_points.npz  the returned points themselves
  ref_c1.json         C1 (generators.random_lp, seed 20261001): instance hash,
                      sha256 of (x, y, Kx, K'y) after each of the first 100
                      iterations of the re-driven loop, D1/D2 and K^T hashes, and
                      the full solve summary at eps 1e-4
  ref_c1_iter100.npz  the iterate after 100 iterations (x, y)
"""
from __future__ import annotations

import glob
import hashlib
import json
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import oracle as O  # noqa: E402
from paper_2311_12180_b200 import SolverParams, generators  # noqa: E402
from paper_2311_12180_b200.lp import GeneralFormLp  # noqa: E402

FIX = Path("/root/reference/proj/tests/fixtures")
OUT = Path(__file__).resolve().parent


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def lp_hash(lp: GeneralFormLp) -> str:
    G, A = lp.inequality_matrix, lp.equality_matrix
    return sha(G.row_offsets, G.col_indices.astype(np.int64), G.values, A.row_offsets,
               A.col_indices.astype(np.int64), A.values, lp.objective, lp.inequality_rhs,
               lp.equality_rhs, lp.lower, lp.upper, np.array([lp.objective_constant]))


def save_lp(path: Path, lp: GeneralFormLp) -> None:
    G, A = lp.inequality_matrix, lp.equality_matrix
    np.savez_compressed(path, g_off=G.row_offsets, g_col=G.col_indices.astype(np.int64), g_val=G.values,
                        a_off=A.row_offsets, a_col=A.col_indices.astype(np.int64), a_val=A.values,
                        c=lp.objective, h=lp.inequality_rhs, b=lp.equality_rhs, l=lp.lower, u=lp.upper,
                        c0=np.array([lp.objective_constant]))


def main() -> None:
    if not O.available("ref"):
        raise SystemExit("build oracle/_ref first: make -C oracle ref")
    (OUT / "suite").mkdir(exist_ok=True)
    files = sorted(glob.glob(str(FIX / "suite" / "*.mps"))) + [
        str(FIX / n) for n in ("infeasible_primal.mps", "infeasible_dual.mps", "tiny2.mps", "objconst.mps")
    ]
    suite = {}
    points = {}
    for f in files:
        name = os.path.basename(f)[:-4]
        lp = O.read_mps(f)
        save_lp(OUT / "suite" / f"{name}.npz", lp)
        limit = 10000 if name.startswith("infeasible") else 1_000_000
        for tag, freq in (("", 64), ("_eager", 1)):
            if freq == 1 and name not in ("twovar", "degen", "prodmix", "rand01", "rand04"):
                continue  # criterion 4 instances (acceptance_main.cpp:187-230)
            p = SolverParams(eps_optimal=1e-8, time_limit_seconds=60.0, iteration_limit=limit,
                             evaluation_frequency=freq, record_step_log=True)
            r = O.solve(lp, p, "ref")
            key = name + tag
            suite[key] = {
                "status": str(r.status), "iterations": r.iterations, "restarts": r.restarts,
                "primal_objective": r.info["primal_objective"], "dual_objective": r.info["dual_objective"],
                "point_sha256": sha(r.point.primal, r.point.dual),
                "lambda_sha256": sha(r.reduced.lambda_),
                "step_log_sha256": sha(r.step_log),
                "restart_log": [[int(e["total_iterations"]), int(e["epoch_length"]), int(e["criterion"]),
                                 int(e["candidate_is_average"]), float(e["omega_after"])] for e in r.restart_log],
                "lp_sha256": lp_hash(lp),
            }
            points[key + "__x"] = r.point.primal
            points[key + "__y"] = r.point.dual
            print(key, suite[key]["status"], r.iterations)
    (OUT / "ref_suite.json").write_text(json.dumps(suite, indent=1, sort_keys=True))
    np.savez_compressed(OUT / "ref_suite_points.npz", **points)

    # ---- C1 ----
    lp = generators.config("C1")
    c1 = {"lp_sha256": lp_hash(lp), "n": lp.num_variables, "m": lp.num_constraints, "nnz": lp.nnz}
    d1, d2 = O.scaling(lp, SolverParams(), "ref")
    c1["scaling_sha256"] = sha(d1, d2)
    from paper_2311_12180_b200.lp import CsrMatrix  # noqa: E402
    K = lp.inequality_matrix
    A = lp.equality_matrix
    nnz_g = K.nnz
    stacked = CsrMatrix(lp.num_constraints, lp.num_variables,
                        np.concatenate([K.row_offsets, A.row_offsets[1:] + nnz_g]),
                        np.concatenate([K.col_indices, A.col_indices]).astype(np.int64),
                        np.concatenate([K.values, A.values]))
    kt = O.transpose(stacked, "ref")
    c1["transpose_sha256"] = sha(kt.row_offsets, kt.col_indices, kt.values)
    s = O.Session(lp, SolverParams(), "ref")
    hashes = []
    for k in range(1, 101):
        s.run(1)
        it = s.iterate()
        hashes.append([it["total"], it["inner"], it["outer"], sha(it["x"], it["y"], it["kx"], it["kty"]),
                       float(it["eta"]), float(it["omega"])])
    np.savez_compressed(OUT / "ref_c1_iter100.npz", x=it["x"], y=it["y"])
    c1["iterates"] = hashes
    r = O.solve(lp, SolverParams(record_step_log=True), "ref")
    c1["solve_1e-4"] = {"status": str(r.status), "iterations": r.iterations, "restarts": r.restarts,
                        "primal_objective": r.info["primal_objective"],
                        "point_sha256": sha(r.point.primal, r.point.dual)}
    (OUT / "ref_c1.json").write_text(json.dumps(c1, indent=1))
    print("C1", c1["solve_1e-4"])


if __name__ == "__main__":
    main()
