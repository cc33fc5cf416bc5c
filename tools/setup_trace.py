"""Setup-phase trace of pdlp_create on a config (dev tool; run on a GPU box):
PDLP_TRACE_SETUP=1 prints per-phase host wall times, this wraps the whole
create and the Python-side conversion.

  python tools/setup_trace.py C4
"""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ["PDLP_TRACE_SETUP"] = "1"
from paper_2311_12180_b200 import Solver, SolverParams, generators  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
lp = generators.config(cfg)
for rep in range(2):
    t0 = time.perf_counter()
    lp.validate()
    tv = time.perf_counter()
    s = Solver(lp, SolverParams())
    t1 = time.perf_counter()
    r = s.solve()
    t2 = time.perf_counter()
    s.close()
    t3 = time.perf_counter()
    print(f"{cfg} #{rep}: validate {1e3 * (tv - t0):.1f} ms, create {1e3 * (t1 - t0):.1f} ms (incl. a second "
          f"validate), solve {1e3 * (t2 - t1):.1f} ms (device {1e3 * r.info['device_seconds']:.1f}), "
          f"close {1e3 * (t3 - t2):.1f} ms", file=sys.stderr, flush=True)
