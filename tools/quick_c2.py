"""Quick timing probe: C2 transportation solve on the GPU (dev tool)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2311_12180_b200 import Solver, SolverParams, generators

for name, lp in (("C1", generators.config("C1")), ("C2", generators.config("C2"))):
    t = time.time()
    s = Solver(lp, SolverParams())
    t_setup = time.time() - t
    for rep in range(3):
        t = time.time()
        r = s.solve()
        dt = time.time() - t
        print(f"{name} setup {t_setup:.3f}s solve {dt:.4f}s status {r.status} it {r.iterations} restarts {r.restarts} "
              f"trials {r.info['trials']} evals {r.info['evaluations']} it/s {r.iterations/dt:.1f} obj {r.info['primal_objective']:.10g}", flush=True)
    for which in (0, 1):
        ms, by = s.time_kernel(which, 50)
        print(f"  kernel {which}: {ms*1e3:.1f} us  {by/1e6:.1f} MB  {by/ms/1e6:.1f} GB/s", flush=True)
    s.close()
