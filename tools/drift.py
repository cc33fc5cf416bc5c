"""Fast-mode drift from the oracle over the first 100 iterates (dev tool):
prints the worst relative distance ||z - z_ref|| / ||z_ref|| per instance."""
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import oracle as O  # noqa: E402  (checker only)
from paper_2311_12180_b200 import Solver, SolverParams, generators  # noqa: E402
from tests.helpers import load_golden_lp  # noqa: E402

CASES = {
    "staircase": lambda: generators.staircase_lp(3, 2000, 500, 500, seed=8),
    "multicommodity": lambda: generators.multicommodity_lp(300, 2000, 5, seed=4),
    "C1": lambda: generators.config("C1"),
    "transport": lambda: generators.transport_lp(60, 80, seed=11),
}
for name in sys.argv[1:] or list(CASES):
    lp = CASES[name]()
    ref = O.Session(lp, SolverParams(), "oracle")
    worst, per = 0.0, []
    with Solver(lp, SolverParams()) as s:
        s.iterate_begin()
        for k in range(100):
            s.iterate_run(1)
            ref.run(1)
            a, b = s.iterate(), ref.iterate()
            za, zb = np.concatenate([a["x"], a["y"]]), np.concatenate([b["x"], b["y"]])
            d = float(np.linalg.norm(za - zb) / max(np.linalg.norm(zb), 1e-300))
            worst = max(worst, d)
            if k in (0, 9, 49, 99) or (os.environ.get("ALL") and k >= 55 and k % 3 == 0):
                per.append(f"{k + 1}:{d:.2e}")
            eta_a, eta_b = a["eta"], b["eta"]
    ref.close()
    print(name, os.environ.get("PDLP_STREAM_NNZ", "auto"), f"worst {worst:.3e}", " ".join(per),
          f"eta rel {abs(eta_a - eta_b) / abs(eta_b):.2e}", flush=True)
