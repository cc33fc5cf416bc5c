cd $GRAFT_REPO_ROOT
timeout 600 python - <<'PY'
import os, sys, time
sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"])
from paper_2311_12180_b200 import Solver, SolverParams, generators
lp = generators.config(os.environ.get("CFG", "C2"))
for k in range(3):
    if k == 2:
        os.environ["PDLP_TRACE_SETUP"] = "1"
    t0 = time.perf_counter(); s = Solver(lp, SolverParams()); t1 = time.perf_counter()
    r = s.solve(); t2 = time.perf_counter(); s.close(); t3 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.2f} ms solve {1e3*(t2-t1):.2f} ms (device {1e3*r.info['device_seconds']:.2f}) close {1e3*(t3-t2):.2f}", flush=True)
PY
