cd $GRAFT_REPO_ROOT
cat > /tmp/c4w.py <<'PY'
import os, sys, time
sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"])
from paper_2311_12180_b200 import Solver, SolverParams, generators
lp = generators.config("C4")
for w in [int(x) for x in sys.argv[1:]]:
    if w > 0:
        os.environ["PDLP_PANELS"] = "1"; os.environ["PDLP_PANEL_WIDTH"] = str(w)
    else:
        os.environ["PDLP_PANELS"] = "0"
    s = Solver(lp, SolverParams(iteration_limit=256))
    r = s.solve()
    d = s.time_kernel(0, 20); p = s.time_kernel(1, 20)
    print(f"width {w}: {r.iterations} it {r.info['device_seconds']:.3f}s -> {r.iterations/r.info['device_seconds']:.1f} it/s; dual {d[0]:.3f} ms primal {p[0]:.3f} ms", flush=True)
    s.close()
PY
timeout 1500 python /tmp/c4w.py 0 3145728 6291456 12582912
