"""Fast vs parity mode on one config (dev tool): iterations, device time, it/s.

  CFG=C2 python tools/parity_speed.py
"""
import os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
from paper_2311_12180_b200 import Solver, SolverParams, generators, Mode
lp = generators.config(os.environ.get("CFG", "C2"))
for mode in (Mode.FAST, Mode.PARITY):
    s = Solver(lp, SolverParams(mode=mode))
    r = s.solve(); r = s.solve()
    print(mode, r.iterations, f"{r.info['device_seconds']*1e3:.1f} ms", f"{r.iterations / r.info['device_seconds']:.0f} it/s", flush=True)
    s.close()
