cd $GRAFT_REPO_ROOT
PDLP_TRACE_SETUP=1 timeout 300 python - <<'PY'
import time
from paper_2311_12180_b200 import Solver, SolverParams, generators
lp = generators.config("C2")
for i in range(3):
    t = time.time(); s = Solver(lp, SolverParams()); t1 = time.time(); s.close(); print("create", 1e3*(t1-t), "destroy", 1e3*(time.time()-t1), flush=True)
PY
