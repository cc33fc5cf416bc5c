cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for c in C1 C2 C3; do echo "=== $c"; ENGINE=2 timeout 300 python tools/micro.py $c 2>&1 | grep -v copy; done
timeout 1200 python /tmp/c4w.py 2>/dev/null || (cat > /tmp/c4w2.py <<PY
import os, sys
sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"])
from paper_2311_12180_b200 import Solver, SolverParams, generators
lp = generators.config("C4")
s = Solver(lp, SolverParams(iteration_limit=256))
r = s.solve()
print("C4", r.iterations / r.info["device_seconds"], "it/s", flush=True)
PY
timeout 1200 python /tmp/c4w2.py)
