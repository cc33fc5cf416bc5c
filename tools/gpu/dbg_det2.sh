cd $GRAFT_REPO_ROOT
cat > /tmp/det.py <<'PY'
import os, sys, numpy as np
sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"])
from paper_2311_12180_b200 import SolverParams, solve
from tests.test_gpu_parity import skewed_lp
lp = skewed_lp()
rs = [solve(lp, SolverParams(eps_optimal=1e-6, iteration_limit=2)) for _ in range(10)]
print(os.environ.get("TAG"), "diffs", [int(np.sum(rs[0].point.primal != r.point.primal)) for r in rs[1:]],
      "kkt", sorted(set(r.info["kkt_omega"] for r in rs)))
PY
TAG="default" timeout 120 python /tmp/det.py
TAG="nofork" PDLP_NO_EVAL_FORK=1 timeout 120 python /tmp/det.py
TAG="smax32" PDLP_STREAM_MAX_ROW=32 timeout 120 python /tmp/det.py
TAG="nofork smax32" PDLP_NO_EVAL_FORK=1 PDLP_STREAM_MAX_ROW=32 timeout 120 python /tmp/det.py
