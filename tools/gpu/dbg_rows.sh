cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cat > /tmp/rows.py <<'PY'
import os, sys, numpy as np
sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"])
from paper_2311_12180_b200 import SolverParams, Solver
from tests.test_gpu_parity import skewed_lp
lp = skewed_lp()
out = {}
with Solver(lp, SolverParams(eps_optimal=1e-6, iteration_limit=4)) as s:
    s.iterate_begin()
    for k in range(4):
        s.iterate_run(1); it = s.iterate()
        for key in ("x", "y", "kx", "kty"):
            out[f"{key}{k}"] = it[key].copy()
        out[f"sc{k}"] = np.array([it["eta"], it["eta_hat"], it["omega"], it["weight_sum"], it["trials"]])
np.savez(f"gpurun_out/rows_{os.environ['TAG']}.npz", **out)
print("saved", os.environ["TAG"])
PY
export PDLP_GRAPH=0
TAG=plain timeout 300 python /tmp/rows.py
TAG=init timeout 900 compute-sanitizer --tool initcheck python /tmp/rows.py 2>&1 | tail -3
TAG=nopdl PDLP_NO_PDL=1 timeout 300 python /tmp/rows.py
TAG=dsep1 PDLP_DECIDE_SEP=1 timeout 300 python /tmp/rows.py
TAG=dsep1init PDLP_DECIDE_SEP=1 timeout 900 compute-sanitizer --tool initcheck python /tmp/rows.py 2>&1 | tail -3
