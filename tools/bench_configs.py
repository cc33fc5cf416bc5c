"""Per-config measurements beside bench.py's headline line:
iterations/s, time to tolerance, and the SpMV / fused-kernel GB/s of every
BASELINE.json configuration on one B200.

  python tools/bench_configs.py C1 C2 C3 C4 [C5] > gpurun_out/configs.jsonl

Per config: setup (upload + K^T build + preconditioning) time; a full solve to
1e-4 (and 1e-8 for C1/C2) under a time limit, reporting status / iterations /
device time; iterations/s over a fixed iteration budget; the four hot kernels
timed with CUDA events on the solver's stream against their algorithmic bytes.
Inputs are generated on the host (seeded); all timing is device-side.
"""
from __future__ import annotations

import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2311_12180_b200 import Solver, SolverParams, generators  # noqa: E402

def _peak() -> float:
    """HBM peak: MEASURED_PEAKS.json (driver-written) when present, else the
    6650 GB/s fallback of B200_PROFILING.md -- the same choice as bench.py."""
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import bench

    return bench.peaks()[0]


PEAK = _peak()
LIMITS = {"C1": 60.0, "C2": 120.0, "C3": 120.0, "C4": 120.0, "C5": 240.0}
FIXED_ITERS = {"C1": 2048, "C2": 2048, "C3": 1024, "C4": 512, "C5": 256}


def b_iter(n: int, m: int, nnz: int) -> float:
    return 24.0 * nnz + 4.0 * (m + n + 2) + 8.0 * (10 * n + 8 * m)


def run(name: str) -> dict:
    t = time.time()
    lp = generators.config(name)
    gen_s = time.time() - t
    n, m, nnz = lp.num_variables, lp.num_constraints, lp.nnz
    out = {"config": name, "n": n, "m": m, "nnz": nnz, "generate_s": gen_s, "b_iter_bytes": b_iter(n, m, nnz)}
    for i, eps in enumerate((1e-4, 1e-8) if name in ("C1", "C2") else (1e-4,)):
        t = time.time()
        s = Solver(lp, SolverParams(eps_optimal=eps, time_limit_seconds=LIMITS[name]))
        if i == 0:
            out["setup_s"] = time.time() - t
        r = s.solve()
        s.close()
        out[f"solve_{eps:g}"] = {"status": str(r.status), "iterations": r.iterations, "restarts": r.restarts,
                                 "device_s": r.info["device_seconds"], "trials": r.info["trials"],
                                 "it_per_s": r.iterations / max(r.info["device_seconds"], 1e-12),
                                 "primal_objective": r.info["primal_objective"],
                                 "relative_gap": r.info["relative_gap"]}
        print(name, eps, out[f"solve_{eps:g}"], file=sys.stderr, flush=True)
    s = Solver(lp, SolverParams(iteration_limit=FIXED_ITERS[name], time_limit_seconds=LIMITS[name]))
    r = s.solve()
    its = r.iterations / max(r.info["device_seconds"], 1e-12)
    out["fixed_iterations"] = {"iterations": r.iterations, "device_s": r.info["device_seconds"], "it_per_s": its,
                               "iteration_gbs": b_iter(n, m, nnz) * its / 1e9,
                               "iteration_frac": b_iter(n, m, nnz) * its / 1e9 / PEAK}
    del lp
    kern = {}
    for which, kname in ((2, "spmv_K"), (3, "spmv_KT"), (0, "dual"), (1, "primal")):
        ms, by = s.time_kernel(which, 50)
        kern[kname] = {"us": 1e3 * ms, "bytes": by, "gbs": by / (ms * 1e-3) / 1e9,
                       "frac": by / (ms * 1e-3) / 1e9 / PEAK}
    out["kernels"] = kern
    s.close()
    return out


def main() -> None:
    for name in sys.argv[1:] or ["C1", "C2", "C3", "C4"]:
        print(json.dumps(run(name)), flush=True)


if __name__ == "__main__":
    main()
