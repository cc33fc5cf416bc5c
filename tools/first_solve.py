"""First and repeated solves on fresh handles (dev tool): create / solve wall
and device time, to see one-time costs (context, module loading, graph
instantiation) land outside the solve's device clock.
"""
import os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
from paper_2311_12180_b200 import Solver, SolverParams, generators
lp = generators.config("C2")
for k in range(3):
    t0 = time.perf_counter(); s = Solver(lp, SolverParams()); t1 = time.perf_counter()
    r = s.solve(); t2 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.1f} ms, solve wall {1e3*(t2-t1):.1f} ms, device {1e3*r.info['device_seconds']:.1f} ms, it {r.iterations}", flush=True)
    s.close()
