cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=graph timeout 300 python /dev/stdin <<'PY'
import os, sys, numpy as np, hashlib
sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"])
from paper_2311_12180_b200 import SolverParams, Solver, solve
from tests.test_gpu_parity import skewed_lp
lp = skewed_lp()
for eng in ("1", "0"):
    os.environ["PDLP_GRAPH"] = eng
    hs = set()
    for _ in range(25):
        with Solver(lp, SolverParams(eps_optimal=1e-6, iteration_limit=2)) as s:
            s.iterate_begin(); s.iterate_run(2); it = s.iterate()
            hs.add(hashlib.md5(it["x"].tobytes() + it["y"].tobytes()).hexdigest()[:8])
    rs = set()
    for _ in range(6):
        r = solve(lp, SolverParams(eps_optimal=1e-6))
        rs.add((r.iterations, hashlib.md5(r.point.primal.tobytes()).hexdigest()[:8]))
    print("graph" if eng == "1" else "stream", "distinct iterates:", hs, "distinct solves:", rs)
PY
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
