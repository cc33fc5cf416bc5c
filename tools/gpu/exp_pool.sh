cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
PDLP_TRACE_SETUP=1 timeout 300 python - <<'PY' 2>&1 | grep -v "pdlp setup" 
import time
from paper_2311_12180_b200 import Solver, SolverParams, generators
lp = generators.config("C2")
for i in range(4):
    t = time.time(); s = Solver(lp, SolverParams()); t1 = time.time(); s.close(); print("create %.1f destroy %.1f ms" % (1e3*(t1-t), 1e3*(time.time()-t1)), flush=True)
PY
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', d['value'], 'e2e', d['e2e'])"
