"""A/B of library variants on one large config without regenerating it per
variant (dev tool): the instance is generated once and kept in /dev/shm as
.npy files; each variant runs in its own process (PDLP_LIB=<variant .so>, plus
optional env vars) and reports a fixed-iteration solve and the hot kernels.

  python tools/ab_config.py C4 base 's3:' 's2:' 'mb40::PDLP_PANEL_MB=40' ...

Variant syntax: name[:defines[:ENV=V,...]] — `defines` selects
lib/variants/<name>.so (tools/build_variants.py); empty means the product lib.
"""
import json
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

CHILD = r'''
import json, os, sys
import numpy as np
sys.path.insert(0, os.environ["ROOT"])
from paper_2311_12180_b200 import Solver, SolverParams
from paper_2311_12180_b200.lp import CsrMatrix, GeneralFormLp
d = os.environ["AB_DIR"]
L = lambda k: np.load(f"{d}/{k}.npy")
n = int(L("c").size)
G = CsrMatrix(int(L("g_off").size) - 1, n, L("g_off"), L("g_col"), L("g_val"))
A = CsrMatrix(int(L("a_off").size) - 1, n, L("a_off"), L("a_col"), L("a_val"))
lp = GeneralFormLp(G, A, L("c"), L("h"), L("b"), L("l"), L("u"))
iters = int(os.environ.get("AB_ITERS", "128"))
s = Solver(lp, SolverParams(iteration_limit=iters, time_limit_seconds=300.0))
r = s.solve(); r = s.solve()
out = {"it_per_s": r.iterations / r.info["device_seconds"]}
for which, name in ((2, "K"), (3, "KT"), (0, "dual"), (1, "primal")):
    ms, by = s.time_kernel(which, 20)
    out[name] = round(ms * 1e3, 1)
print(json.dumps(out))
'''


def main() -> None:
    from paper_2311_12180_b200 import generators

    cfg, specs = sys.argv[1], sys.argv[2:]
    d = Path(f"/dev/shm/ab_{cfg}")
    d.mkdir(parents=True, exist_ok=True)
    t = time.time()
    lp = generators.config(cfg)
    G, A = lp.inequality_matrix, lp.equality_matrix
    for k, v in {"g_off": G.row_offsets, "g_col": G.col_indices, "g_val": G.values, "a_off": A.row_offsets,
                 "a_col": A.col_indices, "a_val": A.values, "c": lp.objective, "h": lp.inequality_rhs,
                 "b": lp.equality_rhs, "l": lp.lower, "u": lp.upper}.items():
        np.save(d / f"{k}.npy", v)
    del lp, G, A
    print(f"# {cfg} staged in {time.time() - t:.0f} s", file=sys.stderr, flush=True)
    for rnd in range(int(os.environ.get("AB_ROUNDS", "1"))):
        for spec in specs:
            name, _, rest = spec.partition(":")
            defs, _, envs = rest.partition(":")
            env = dict(os.environ, ROOT=str(ROOT), AB_DIR=str(d))
            so = ROOT / "paper_2311_12180_b200" / "lib" / "variants" / f"{name}.so"
            if defs and so.exists():
                env["PDLP_LIB"] = str(so)
            for kv in filter(None, envs.split(",")):
                k, _, v = kv.partition("=")
                env[k] = v
            r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
            line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else json.dumps({"error": r.stderr[-500:]})
            print(json.dumps({"variant": spec, "round": rnd, **json.loads(line)}), flush=True)


if __name__ == "__main__":
    main()
