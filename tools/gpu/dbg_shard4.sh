cd $GRAFT_REPO_ROOT
timeout 600 python - <<'PY'
import numpy as np
from paper_2311_12180_b200 import ShardGroup, SolverParams, solve
from tests.test_gpu_parity import skewed_lp
lp = skewed_lp()
p = SolverParams(eps_optimal=1e-6, iteration_limit=2)
with ShardGroup(lp, p, 2) as g:
    res = g.solve()
a = res[0]
for pw in (0, 2, 3):
    b = solve(lp, SolverParams(eps_optimal=1e-6, iteration_limit=2, plan_world=pw))
    print("plan_world", pw, "x diff", int(np.sum(a.point.primal != b.point.primal)), "y diff", int(np.sum(a.point.dual != b.point.dual)))
b1 = solve(lp, SolverParams(eps_optimal=1e-6, iteration_limit=2, plan_world=2))
b2 = solve(lp, SolverParams(eps_optimal=1e-6, iteration_limit=2, plan_world=2))
print("plan_world repeat x diff", int(np.sum(b1.point.primal != b2.point.primal)))
with ShardGroup(lp, p, 2) as g:
    res2 = g.solve()
print("shard repeat x diff", int(np.sum(res2[0].point.primal != a.point.primal)), "rank1 vs rank0", int(np.sum(res2[1].point.primal != res2[0].point.primal)))
PY
