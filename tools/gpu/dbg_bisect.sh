cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cat > /tmp/bis.py <<'PY'
import os, sys, numpy as np, hashlib
sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"])
from paper_2311_12180_b200 import SolverParams, Solver
from tests.test_gpu_parity import skewed_lp
lp = skewed_lp()
with Solver(lp, SolverParams(eps_optimal=1e-6, iteration_limit=2)) as s:
    s.iterate_begin(); s.iterate_run(int(os.environ.get("NIT", "2"))); it = s.iterate()
np.savez(f"gpurun_out/bis_{os.environ['TAG']}.npz", x=it["x"], y=it["y"], kx=it["kx"], kty=it["kty"])
print(os.environ["TAG"], hashlib.md5(it["x"].tobytes() + it["y"].tobytes()).hexdigest()[:8], it["trials"])
PY
export PDLP_GRAPH=0
run() { tag=$1; shift; env "$@" TAG=${tag}_p timeout 300 python /tmp/bis.py; env "$@" TAG=${tag}_i timeout 900 compute-sanitizer --tool initcheck python /tmp/bis.py 2>&1 | grep -v "=====" ; }
run base X=1
run nopdl PDLP_NO_PDL=1
run nolazy PDLP_NO_LAZY_KTY=1
run s32 PDLP_STREAM_MAX_ROW=32
run s64 PDLP_STREAM_MAX_ROW=64
run nogrp PDLP_NO_ROW_GROUPS=1
run dsep1 PDLP_DECIDE_SEP=1
run nofork PDLP_NO_EVAL_FORK=1
run n3 NIT=3
