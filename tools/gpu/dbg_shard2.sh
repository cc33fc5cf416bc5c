cd $GRAFT_REPO_ROOT
timeout 600 python - <<'PY'
import threading, numpy as np
from paper_2311_12180_b200 import ShardGroup, SolverParams, Solver
from tests.test_gpu_parity import skewed_lp
lp = skewed_lp()
p = SolverParams(eps_optimal=1e-6, iteration_limit=20000)
g = ShardGroup(lp, p, 2)
ref = Solver(lp, SolverParams(eps_optimal=1e-6, iteration_limit=20000, plan_world=2))
def par(fn):
    ts=[threading.Thread(target=fn, args=(r,)) for r in g.ranks]
    [t.start() for t in ts]; [t.join() for t in ts]
par(lambda r: r.iterate_begin()); ref.iterate_begin()
info = [r.shard_info() for r in g.ranks]; print(info)
for k in range(1, 70):
    par(lambda r: r.iterate_run(1)); ref.iterate_run(1)
    a = g.ranks[0].iterate(); b = ref.iterate()
    dx = np.nonzero(a["x"] != b["x"])[0]; dy = np.nonzero(a["y"] != b["y"])[0]
    if len(dx) or len(dy) or a["eta"] != b["eta"] or a["omega"] != b["omega"]:
        print("k", k, "total", a["total"], b["total"], "dx", len(dx), dx[:8], "dy", len(dy), dy[:8], "eta", a["eta"], b["eta"], "omega", a["omega"], b["omega"])
        kx0 = g.ranks[0].iterate()["kx"]; kxr = b["kx"]
        r0, r1 = info[0]["row0"], info[0]["row1"]
        print("  kx own diff", np.nonzero(kx0[r0:r1] != kxr[r0:r1])[0][:8])
        break
else:
    print("no diff in 69 iterations")
PY
