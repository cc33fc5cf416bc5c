cd $GRAFT_REPO_ROOT
timeout 600 python - <<'PY'
import numpy as np
from paper_2311_12180_b200 import ShardGroup, SolverParams, solve
from tests.test_gpu_parity import skewed_lp
lp = skewed_lp()
p = SolverParams(eps_optimal=1e-6, iteration_limit=20000)
for w in (2, 3):
    with ShardGroup(lp, p, w) as g:
        res = g.solve()
    ref = solve(lp, SolverParams(eps_optimal=1e-6, iteration_limit=20000, plan_world=w))
    a, b = res[0], ref
    print("world", w, a.status, b.status, a.iterations, b.iterations, a.restarts, b.restarts)
    for name, u, v in (("x", a.point.primal, b.point.primal), ("y", a.point.dual, b.point.dual), ("lam", a.reduced.lambda_, b.reduced.lambda_)):
        d = np.nonzero(u != v)[0]
        print("  ", name, len(d), d[:10], np.max(np.abs(u - v)) if len(d) else 0)
    print("   obj", a.info["primal_objective"], b.info["primal_objective"])
PY
