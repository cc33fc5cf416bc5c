"""Panel-geometry probe (dev tool; run under ncu for DRAM bytes, numbers
printed here come from CUDA events). One process: the config is generated
once, then for each variant (name:ENV=V,ENV=V) the environment is set, a
Solver is created (build_panels reads the knobs at create time), and the two
plain panel SpMVs are timed: K x (2) and K^T y (3).

  python tools/panel_probe.py C4 base: b16:PDLP_BAND_MB=16 ...
"""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2311_12180_b200 import Solver, SolverParams, generators  # noqa: E402

KNOBS = ("PDLP_PANELS", "PDLP_PANEL_MB", "PDLP_BAND_MB", "PDLP_PANEL_MB_K", "PDLP_PANEL_MB_T", "PDLP_BAND_MB_K",
         "PDLP_BAND_MB_T", "PDLP_PANEL_WORKERS", "PDLP_PANEL_MIN_MB")
cfg = sys.argv[1]
lp = generators.config(cfg)
reps = int(os.environ.get("PROBE_REPS", "3"))
for spec in sys.argv[2:]:
    name, _, envs = spec.partition(":")
    for k in KNOBS:
        os.environ.pop(k, None)
    for kv in filter(None, envs.split(",")):
        k, _, v = kv.partition("=")
        os.environ[k] = v
    with Solver(lp, SolverParams(iteration_limit=1)) as s:
        out = {"variant": spec}
        for w, nm in ((2, "K"), (3, "KT")):
            ms, _ = s.time_kernel(w, reps)
            kb = s.kernel_bytes(w)
            out[nm] = {"us": round(ms * 1e3, 1), "panels": kb["panels"], "bands": kb["bands"]}
        print(json.dumps(out), flush=True)
