"""Profiling driver: one warm C2 solve (run under ncu; numbers printed here are not bench values).
Graph replay is disabled (ncu cannot profile kernel nodes of graphs with conditional nodes)."""
import os
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2311_12180_b200 import Solver, SolverParams, generators

which = sys.argv[1] if len(sys.argv) > 1 else "C2"
lp = generators.config(which)
limit = int(os.environ.get("PDLP_ITER_LIMIT", str(2**62)))
s = Solver(lp, SolverParams(use_cuda_graph=os.environ.get("PDLP_GRAPH", "0") == "1", iteration_limit=limit))
r = s.solve()
print(which, r.status, r.iterations, r.info["device_seconds"])
s.close()
