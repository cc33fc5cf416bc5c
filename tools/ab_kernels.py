"""A/B timing of the hot kernels across library variants (dev tool).

  python tools/ab_kernels.py C2 base shift16 'contig:PDLP_CONTIG=1' ...

A variant is `name[:ENV=V,ENV2=V2]`: lib/variants/<name>.so when that exists
(tools/build_variants.py), else the product library, run with those env vars.

Per variant: the four hot kernels (CUDA events, 200 launches) and a solve's
device time; interleaved rounds so clock drift hits every variant alike."""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
CHILD = r'''
import json, os, sys
sys.path.insert(0, os.environ["ROOT"])
from paper_2311_12180_b200 import Solver, SolverParams, generators
lp = generators.config(os.environ["CFG"])
s = Solver(lp, SolverParams(engine=int(os.environ.get("AB_ENGINE", "0"))))
r = s.solve(); r = s.solve()
out = {"iters": r.iterations, "solve_ms": r.info["device_seconds"] * 1e3,
       "eval_ms": r.info["eval_seconds"] * 1e3, "window_ms": r.info["window_seconds"] * 1e3}
for which, name in ((2, "K"), (3, "KT"), (0, "dual"), (1, "primal")):
    ms, by = s.time_kernel(which, 200)
    out[name] = round(ms * 1e3, 2)
print(json.dumps(out))
'''

cfg, variants = sys.argv[1], sys.argv[2:]
rounds = int(os.environ.get("ROUNDS", "3"))
res = {v: [] for v in variants}
for _ in range(rounds):
    for v in variants:
        name, _, envs = v.partition(":")
        env = dict(os.environ, ROOT=str(ROOT), CFG=cfg)
        lib = ROOT / "paper_2311_12180_b200" / "lib" / "variants" / f"{name}.so"
        if lib.exists():
            env["PDLP_LIB"] = str(lib)
        env.update(kv.split("=", 1) for kv in envs.split(",") if kv)
        p = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, timeout=900)
        if p.returncode:
            print(v, "FAILED", p.stderr[-2000:], flush=True)
            continue
        res[v].append(json.loads(p.stdout.strip().splitlines()[-1]))
for v, rs in res.items():
    if not rs:
        continue
    best = {k: min(r[k] for r in rs) for k in rs[0]}
    print(cfg, v, json.dumps(best), flush=True)
