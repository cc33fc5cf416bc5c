"""Golden vectors of the BASELINE.json configurations from the REFERENCE
solver (oracle/_ref, the unmodified pdhglp headers built by oracle/Makefile).
Run in the build container only (the GPU box has no /root/reference):

    make -C oracle ref && python tests/golden/make_golden_configs.py [C2 C3 C4]

Outputs (committed), per config, configs_<name>.npz + an entry in
configs.json:
  * the instance hash (generators.config(name) is seeded and deterministic);
  * the first N iterates of the re-driven SolveLoop::run (solver.hpp:759-929;
    N = 100 for C2 and C3, 20 for C4): counters (total, inner, trials), eta,
    eta_hat, omega, the 2-norm and max-norm of x and y, and the values of x
    and y at a fixed seeded sample of indices (full vectors are 8-320 MB per
    iterate);
  * C2 only: the reference's full solve at eps 1e-4 and 1e-8 (solve(),
    solver.hpp:935-940): status, iterations, restarts, objectives.

    python tests/golden/make_golden_configs.py --reorder-drift [C2 C3 C4]
    python tests/golden/make_golden_configs.py --solve C3 C4

--solve adds the reference's own full solve at eps 1e-4 (solve(),
solver.hpp:935-940; hours on one core for C4) to each entry: status,
iterations, restarts, objectives.

    python tests/golden/make_golden_configs.py --reorder-drift [C2 C3 C4]

adds `reorder_drift` to each entry: how far the reference's own first N
iterates move when only the summation order of the step-size sums (dx^2, dy^2,
interaction; solver.hpp:422-435) changes from sequential to pairwise trees.
It is measured on the C restatement (oracle/, pinned bitwise to the
reference), with the worst relative error over the N iterates in the 2-norm
and max-norm, over z = (x, y), x and y, as tests/test_gpu_configs.py measures
fast mode. This is the floor any order other than the reference's own
sequential one can reach.
"""
from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import oracle as O  # noqa: E402
from paper_2311_12180_b200 import SolverParams, generators  # noqa: E402
from tests.helpers import lp_hash  # noqa: E402

OUT = Path(__file__).resolve().parent
ITERATES = {"C2": 100, "C3": 100, "C4": 20}
SAMPLES = 16384
SAMPLE_SEED = 20261017
# C2 and C3 are compared against a live reference session on full vectors;
# their goldens only pin that session, so they keep every 8th sample
SAMPLE_STRIDE = {"C2": 8, "C3": 8, "C4": 1}


def sample_indices(size: int, seed: int) -> np.ndarray:
    if size <= SAMPLES:
        return np.arange(size, dtype=np.int64)
    return np.sort(np.random.default_rng(seed).choice(size, SAMPLES, replace=False)).astype(np.int64)


def iterates(name: str, lp) -> dict:
    n, m = lp.num_variables, lp.num_constraints
    st = SAMPLE_STRIDE[name]
    ix, iy = sample_indices(n, SAMPLE_SEED)[::st], sample_indices(m, SAMPLE_SEED + 1)[::st]
    t = time.time()
    s = O.Session(lp, SolverParams(), "ref")
    print(f"{name}: reference setup {time.time() - t:.1f} s", flush=True)
    N = ITERATES[name]
    rec = {k: [] for k in ("total", "inner", "trials", "eta", "eta_hat", "omega", "x_norm", "y_norm", "x_max",
                           "y_max", "x_s", "y_s")}
    t = time.time()
    for _ in range(N):
        s.run(1)
        it = s.iterate()
        for k in ("total", "inner", "trials", "eta", "eta_hat", "omega"):
            rec[k].append(it[k])
        rec["x_norm"].append(np.linalg.norm(it["x"]))
        rec["y_norm"].append(np.linalg.norm(it["y"]))
        rec["x_max"].append(np.abs(it["x"]).max())
        rec["y_max"].append(np.abs(it["y"]).max())
        rec["x_s"].append(it["x"][ix])
        rec["y_s"].append(it["y"][iy])
    s.close()
    print(f"{name}: {N} iterates in {time.time() - t:.1f} s", flush=True)
    out = {k: np.asarray(v) for k, v in rec.items()}
    out["ix"], out["iy"] = ix, iy
    return out


def reorder_drift(name: str, lp) -> dict:
    """The two runs go one after the other (C4's sessions take ~35 GB of host
    memory each); the sequential run's iterates are parked on disk."""
    import tempfile

    N = ITERATES[name]
    n, m = lp.num_variables, lp.num_constraints
    with tempfile.TemporaryDirectory(dir="/root") as tmp:
        store = np.lib.format.open_memmap(f"{tmp}/z.npy", mode="w+", dtype=np.float64, shape=(N, n + m))
        counters = []
        O.set_sum_order(0)
        a = O.Session(lp, SolverParams(), "oracle")
        for k in range(N):
            a.run(1)
            ia = a.iterate()
            store[k, :n], store[k, n:] = ia["x"], ia["y"]
            counters.append((ia["total"], ia["trials"]))
        a.close()
        del a
        w2 = wi = 0.0
        O.set_sum_order(1)
        try:
            b = O.Session(lp, SolverParams(), "oracle")
            for k in range(N):
                b.run(1)
                ib = b.iterate()
                assert (ib["total"], ib["trials"]) == counters[k]
                za = np.asarray(store[k])
                zb = np.concatenate([ib["x"], ib["y"]])
                for u, v in ((za, zb), (za[:n], ib["x"]), (za[n:], ib["y"])):
                    w2 = max(w2, float(np.linalg.norm(v - u) / max(np.linalg.norm(u), 1e-300)))
                    wi = max(wi, float(np.abs(v - u).max(initial=0.0) / max(np.abs(u).max(initial=0.0), 1e-300)))
            b.close()
        finally:
            O.set_sum_order(0)
        del store
    return {"rel2": w2, "relinf": wi, "iterates": N, "order": "pairwise step-size sums (oracle, sum order 1)"}


def main() -> None:
    args = sys.argv[1:]
    if args and args[0] == "--reorder-drift":
        names = args[1:] or ["C2", "C3", "C4"]
        meta_path = OUT / "configs.json"
        meta = json.loads(meta_path.read_text())
        for name in names:
            t = time.time()
            lp = generators.config(name)
            assert lp_hash(lp) == meta[name]["instance_sha256"]
            meta[name]["reorder_drift"] = reorder_drift(name, lp)
            print(f"{name}: {meta[name]['reorder_drift']} ({time.time() - t:.0f} s)", flush=True)
            meta_path.write_text(json.dumps(meta, indent=1, sort_keys=True) + "\n")
            del lp
        return
    if args and args[0] == "--solve":
        meta_path = OUT / "configs.json"
        for name in args[1:]:
            lp = generators.config(name)
            meta = json.loads(meta_path.read_text())
            assert lp_hash(lp) == meta[name]["instance_sha256"]
            t = time.time()
            r = O.solve(lp, SolverParams(eps_optimal=1e-4, time_limit_seconds=1e9), "ref")
            meta = json.loads(meta_path.read_text())  # re-read: other runs may have written meanwhile
            meta[name]["solve_0.0001"] = {"status": str(r.status), "iterations": r.iterations,
                                          "restarts": r.restarts, "primal_objective": r.info["primal_objective"],
                                          "dual_objective": r.info["dual_objective"], "seconds": time.time() - t}
            print(f"{name}: {meta[name]['solve_0.0001']}", flush=True)
            meta_path.write_text(json.dumps(meta, indent=1, sort_keys=True) + "\n")
            del lp
        return
    names = args or ["C2", "C3", "C4"]
    meta_path = OUT / "configs.json"
    meta = json.loads(meta_path.read_text()) if meta_path.exists() else {}
    for name in names:
        t = time.time()
        lp = generators.config(name)
        entry = {"instance_sha256": lp_hash(lp), "n": lp.num_variables, "m": lp.num_constraints,
                 "nnz": lp.nnz, "seed": generators.SEEDS[name], "iterates": ITERATES[name]}
        print(f"{name}: generated in {time.time() - t:.1f} s", flush=True)
        np.savez_compressed(OUT / f"configs_{name}.npz", **iterates(name, lp))
        if name == "C2":
            for eps in (1e-4, 1e-8):
                t = time.time()
                r = O.solve(lp, SolverParams(eps_optimal=eps), "ref")
                entry[f"solve_{eps:g}"] = {"status": str(r.status), "iterations": r.iterations,
                                           "restarts": r.restarts,
                                           "primal_objective": r.info["primal_objective"],
                                           "dual_objective": r.info["dual_objective"],
                                           "seconds": time.time() - t}
                print(f"{name}: solve {eps:g}: {entry[f'solve_{eps:g}']}", flush=True)
        meta[name] = entry
        meta_path.write_text(json.dumps(meta, indent=1, sort_keys=True) + "\n")
        del lp


if __name__ == "__main__":
    main()
