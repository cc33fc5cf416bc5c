cd $GRAFT_REPO_ROOT
cat > /tmp/det.py <<'PY'
import os, sys, numpy as np
sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"])
from paper_2311_12180_b200 import SolverParams, solve, abi
from tests.test_gpu_parity import skewed_lp
lp = skewed_lp()
eng = int(os.environ.get("ENG", "0"))
xs = [solve(lp, SolverParams(eps_optimal=1e-6, iteration_limit=int(os.environ.get("IT", "2")), engine=eng)).point.primal for _ in range(4)]
print(os.environ.get("TAG"), "diffs", [int(np.sum(xs[0] != x)) for x in xs[1:]])
PY
for smax in 32 64; do for eng in 2 3; do for it in 1 2; do TAG="smax=$smax eng=$eng it=$it" PDLP_STREAM_MAX_ROW=$smax ENG=$eng IT=$it timeout 120 python /tmp/det.py; done; done; done
TAG="smax=64 decide1" PDLP_STREAM_MAX_ROW=64 PDLP_DECIDE_SEP=1 ENG=3 timeout 120 python /tmp/det.py
TAG="smax=64 nolazy" PDLP_STREAM_MAX_ROW=64 PDLP_NO_LAZY_KTY=1 ENG=3 timeout 120 python /tmp/det.py
