cd $GRAFT_REPO_ROOT
cat > /tmp/san.py <<'PY'
import os, sys, numpy as np, hashlib
sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"])
from paper_2311_12180_b200 import SolverParams, Solver
from tests.test_gpu_parity import skewed_lp
lp = skewed_lp()
n = int(os.environ.get("REPS", "1"))
hs = []
for _ in range(n):
    with Solver(lp, SolverParams(eps_optimal=1e-6, iteration_limit=2)) as s:
        s.iterate_begin(); s.iterate_run(2); it = s.iterate()
        hs.append(hashlib.md5(it["x"].tobytes() + it["y"].tobytes()).hexdigest()[:8])
print(os.environ.get("TAG"), hs)
PY
TAG=stream REPS=12 PDLP_GRAPH=0 timeout 300 python /tmp/san.py
TAG=graph REPS=12 timeout 300 python /tmp/san.py
export PDLP_GRAPH=0
for tool in initcheck racecheck memcheck; do
  echo "== $tool"
  TAG=$tool timeout 900 compute-sanitizer --tool $tool --print-limit 20 python /tmp/san.py 2>&1 | grep -v "^=========     " | head -60
done
