import os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import ctypes as C
from paper_2311_12180_b200 import Solver, SolverParams, generators, abi
from paper_2311_12180_b200.api import _check
lp = generators.config("C2")
for k in range(3):
    s = Solver(lp, SolverParams())
    info = abi.PdlpResultInfo()
    t0 = time.perf_counter()
    _check(s._lib.pdlp_solve(s._h, C.byref(info)))
    t1 = time.perf_counter()
    s.last_info = info
    r = s.result()
    t2 = time.perf_counter()
    s.close()
    print(f"pdlp_solve {1e3*(t1-t0):.2f} ms (device {1e3*info.device_seconds:.2f}, solve_seconds {1e3*info.solve_seconds:.2f}) result() {1e3*(t2-t1):.2f} ms", flush=True)
