"""Profiling driver (run under ncu; numbers printed here are not bench values):
builds the solver for a config and launches the hot kernels through
pdlp_time_kernel: 0 dual, 1 primal, 2 SpMV K, 3 SpMV K^T.

  ncu ... python tools/ncu_kernels.py C4 2 3
"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2311_12180_b200 import Solver, SolverParams, generators  # noqa: E402

cfg = sys.argv[1]
which = [int(w) for w in sys.argv[2:]] or [0, 1, 2, 3]
lp = generators.config(cfg)
with Solver(lp, SolverParams(iteration_limit=8)) as s:
    del lp
    if os.environ.get("NCU_SOLVE", "1") == "1":
        s.solve()
    for w in which:
        ms, _ = s.time_kernel(w, 1)
        print(cfg, w, f"{ms:.3f} ms")
