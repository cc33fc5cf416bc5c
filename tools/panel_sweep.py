"""A/B of the column-panel budget on one config (default C4): for each
PDLP_PANEL_MB value, setup, a fixed-iteration solve (it/s) and the four hot
kernels timed with CUDA events against their algorithmic and moved bytes.

  python tools/panel_sweep.py [config] [mb ...] > gpurun_out/panel_sweep.jsonl
"""
from __future__ import annotations

import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from bench import b_iter, peaks  # noqa: E402
from paper_2311_12180_b200 import Solver, SolverParams, generators  # noqa: E402


def main() -> None:
    name = sys.argv[1] if len(sys.argv) > 1 else "C4"
    budgets = sys.argv[2:] or ["48"]
    t = time.time()
    lp = generators.config(name)
    print(f"generated {name} in {time.time() - t:.1f} s", file=sys.stderr, flush=True)
    n, m, nnz = lp.num_variables, lp.num_constraints, lp.nnz
    peak = peaks()[0]
    iters = int(os.environ.get("SWEEP_ITERS", "256"))
    for mb in budgets:
        if mb == "off":
            os.environ["PDLP_PANELS"] = "0"
        else:
            os.environ.pop("PDLP_PANELS", None)
            os.environ["PDLP_PANEL_MB"] = mb
        t = time.time()
        s = Solver(lp, SolverParams(iteration_limit=iters, time_limit_seconds=300.0))
        setup = time.time() - t
        r = s.solve()
        its = r.iterations / max(r.info["device_seconds"], 1e-12)
        out = {"config": name, "panel_mb": mb, "setup_s": setup, "iterations": r.iterations,
               "device_s": r.info["device_seconds"], "it_per_s": its,
               "iteration_frac": b_iter(n, m, nnz) * its / 1e9 / peak}
        kern = {}
        for which, kname in ((2, "spmv_K"), (3, "spmv_KT"), (0, "dual"), (1, "primal")):
            ms, alg = s.time_kernel(which, 20)
            kb = s.kernel_bytes(which)
            kern[kname] = {"us": 1e3 * ms, "alg_bytes": alg, "moved_bytes": kb["moved"], "panels": kb["panels"],
                           "alg_frac": alg / (ms * 1e-3) / 1e9 / peak,
                           "moved_frac": kb["moved"] / (ms * 1e-3) / 1e9 / peak}
        out["kernels"] = kern
        s.close()
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
