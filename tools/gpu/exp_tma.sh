cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for c in C1 C2 C3; do echo "=== $c"; ENGINE=2 timeout 300 python tools/micro.py $c 2>&1 | grep -v copy; done
cat > /tmp/c4w.py <<PY
import os, sys
sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"])
from paper_2311_12180_b200 import Solver, SolverParams, generators
lp = generators.config("C4")
for v in ("1", "0"):
    os.environ["PDLP_PANELS"] = v
    s = Solver(lp, SolverParams(iteration_limit=256))
    r = s.solve()
    d = s.time_kernel(0, 20); p = s.time_kernel(1, 20)
    print("panels", v, r.iterations / r.info["device_seconds"], "it/s dual", d[0], "primal", p[0], flush=True)
    s.close()
PY
timeout 1500 python /tmp/c4w.py
