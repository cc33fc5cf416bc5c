cd $GRAFT_REPO_ROOT
cat > /tmp/det3.py <<'PY'
import os, sys, numpy as np
sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"])
from paper_2311_12180_b200 import SolverParams, Solver, solve
from tests.test_gpu_parity import skewed_lp
lp = skewed_lp()
its = []
for _ in range(40):
    with Solver(lp, SolverParams(eps_optimal=1e-6, iteration_limit=2)) as s:
        s.iterate_begin(); s.iterate_run(2); it = s.iterate()
        its.append((it["x"].copy(), it["y"].copy(), it["kx"].copy(), it["kty"].copy()))
print("iterate diffs x,y,kx,kty:", [tuple(int(np.sum(a != b)) for a, b in zip(its[0], t)) for t in its[1:]])
rs = [solve(lp, SolverParams(eps_optimal=1e-6, iteration_limit=2)) for _ in range(40)]
base = rs[0]
for r in rs[1:]:
    d = np.nonzero(r.point.primal != base.point.primal)[0]
    if len(d):
        print("solve differs at", len(d), "entries; y diff", int(np.sum(r.point.dual != base.point.dual)),
              "lam diff", int(np.sum(r.reduced.lambda_ != base.reduced.lambda_)), "iters", r.iterations, base.iterations,
              "sample", d[:5], r.point.primal[d[:3]], base.point.primal[d[:3]],
              "vs iterate x", int(np.sum(r.point.primal != its[0][0])), int(np.sum(base.point.primal != its[0][0])))
PY
timeout 300 python /tmp/det3.py
