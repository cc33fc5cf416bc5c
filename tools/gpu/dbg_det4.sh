cd $GRAFT_REPO_ROOT
cat > /tmp/det4.py <<'PY'
import os, sys, numpy as np
sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"])
from paper_2311_12180_b200 import SolverParams, Solver
from tests.test_gpu_parity import skewed_lp
lp = skewed_lp()
its = []
for _ in range(40):
    with Solver(lp, SolverParams(eps_optimal=1e-6, iteration_limit=2)) as s:
        s.iterate_begin(); s.iterate_run(2); it = s.iterate()
        its.append(it["x"].copy())
print(os.environ.get("TAG"), "runs differing:", sum(int(np.any(its[0] != t)) for t in its[1:]), "of", len(its) - 1)
PY
TAG=default timeout 300 python /tmp/det4.py
TAG=nopdl PDLP_NO_PDL=1 timeout 300 python /tmp/det4.py
TAG=nofork PDLP_NO_EVAL_FORK=1 timeout 300 python /tmp/det4.py
TAG=stream PDLP_GRAPH=0 timeout 300 python /tmp/det4.py
