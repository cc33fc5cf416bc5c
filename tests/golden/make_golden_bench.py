"""Regenerates tests/golden/bench_golden.json from the REFERENCE's benchmark
harness (pdhglp/bench.hpp through oracle/_ref, built from /root/reference by
oracle/Makefile). Run in the build container only:

    make -C oracle ref && python tests/golden/make_golden_bench.py

Contents (committed; the GPU box has no /root/reference):
  hashes    config_hash for several parameter sets and time limits (bench.hpp:135-155)
  sgm       shifted_geometric_mean on fixed lists (bench.hpp:29-41)
  report    write_report of a fixed synthetic record set (bench.hpp:242-262)
  run       the reference's run_benchmark over the golden suite written back
            as MPS (tests.helpers.write_free_mps), eps 1e-4, time limit 60 s:
            per instance nonzeros / status / iterations / objective, and the
            aggregate rows' instance and solved counts (timings vary)
"""
from __future__ import annotations

import ctypes as C
import json
import math
import sys
import tempfile
from dataclasses import replace
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import oracle as O  # noqa: E402
from paper_2311_12180_b200 import SolverParams  # noqa: E402
from paper_2311_12180_b200.lp import ScalingMode  # noqa: E402
from tests.helpers import load_golden_lp, suite_names, write_free_mps  # noqa: E402

OUT = Path(__file__).resolve().parent / "bench_golden.json"

PARAM_SETS = {
    "default": SolverParams(),
    "eps8": SolverParams(eps_optimal=1e-8),
    "limit1000": SolverParams(iteration_limit=1000),
    "no_scaling": SolverParams(scaling=ScalingMode.NONE),
    "theta03_omega1e6": SolverParams(theta_smoothing=0.3, omega_max=1e6),
    "freq32_ruiz5": SolverParams(evaluation_frequency=32, ruiz_iterations=5, pock_chambolle_alpha=0.5),
}
TIME_LIMITS = [60.0, 3600.0, 0.1, 1e-3]

SGM_CASES = [[0.0], [1.0, 2.0, 3.0], [0.5, 100.0, 3600.0, 7.25], [1e-6] * 5, [10.0, 10.0]]

# (instance, nonzeros, parse_failed, status, solve_s, total_s, iterations, obj, gap, rpr, rdr)
RECORDS = [
    ("a_small.mps", 12, 0, 0, 0.25, 0.5, 960, 1.0 / 3.0, 2.5e-5, 1e-6, 3e-7),
    ("b_parse.mps", 0, 1, 5, 0.0, 0.0, 0, 0.0, 0.0, 0.0, 0.0),
    ("c_medium.mps", 1_000_000, 0, 1, 12.5, 13.0, 4096, -0.0, 1.0, 0.5, 0.25),
    ("d_large.mps", 10_000_000, 0, 3, 60.0, 61.5, 100000, 123456789.123, 1e-3, 2e-2, 3e-1),
    ("e_limit.mps", 999_999, 0, 4, 75.0, 76.0, 5, float("inf"), float("inf"), 0.0, 1e300),
    ("f_dual.mps", 20, 0, 2, 0.001, 0.002, 64, -5.5, 0.0, 0.0, 0.0),
    ("g_numerr.mps", 9_999_999, 0, 5, 3.0, 3.5, 7, 1e-320, 5e-324, 0.0, 0.0),
]


def lib():
    L = O.load("ref")
    PP = C.POINTER(O.abi.PdlpParams)
    dp, i64p, i32p = C.POINTER(C.c_double), C.POINTER(C.c_int64), C.POINTER(C.c_int32)
    L.ref_bench_config_hash.argtypes = [PP, C.c_double, C.c_char_p]
    L.ref_bench_sgm.argtypes = [dp, C.c_int64, C.c_double, dp]
    L.ref_bench_report.argtypes = [C.c_int64, C.c_char_p, i64p, i32p, i32p, dp, dp, i64p, dp, dp, dp, dp,
                                   PP, C.c_double, C.c_char_p, C.c_int64, i64p]
    L.ref_bench_run.argtypes = [C.c_char_p, PP, C.c_double, C.c_int32, C.c_char_p, C.c_int64, i64p]
    return L


def ref_hash(L, p: SolverParams, tl: float) -> str:
    buf = C.create_string_buffer(17)
    L.ref_bench_config_hash(C.byref(p.to_abi()), tl, buf)
    return buf.value.decode()


def text_call(fn, *args) -> str:
    cap = 1 << 20
    buf = C.create_string_buffer(cap)
    n = C.c_int64(0)
    rc = fn(*args, buf, cap, C.byref(n))
    if rc != 0:
        raise RuntimeError(f"reference call failed: {rc}")
    return buf.value.decode()


def arr(ctype, vals):
    return (ctype * len(vals))(*vals)


def main() -> None:
    L = lib()
    out = {"hashes": [], "sgm": [], "records": RECORDS}
    for name, p in PARAM_SETS.items():
        for tl in TIME_LIMITS:
            out["hashes"].append({"params": name, "time_limit": tl, "hash": ref_hash(L, p, tl)})
    for ts in SGM_CASES:
        v = C.c_double(0.0)
        assert L.ref_bench_sgm(arr(C.c_double, ts), len(ts), 10.0, C.byref(v)) == 0
        out["sgm"].append({"times": ts, "shift": 10.0, "value": v.value})
    cols = list(zip(*RECORDS))
    names = "\n".join(cols[0]).encode()
    p = SolverParams()
    out["report"] = text_call(
        L.ref_bench_report, len(RECORDS), names, arr(C.c_int64, cols[1]), arr(C.c_int32, cols[2]),
        arr(C.c_int32, cols[3]), arr(C.c_double, cols[4]), arr(C.c_double, cols[5]), arr(C.c_int64, cols[6]),
        arr(C.c_double, cols[7]), arr(C.c_double, cols[8]), arr(C.c_double, cols[9]), arr(C.c_double, cols[10]),
        C.byref(p.to_abi()), 60.0)
    # the reference's directory benchmark over the suite, written back as MPS
    with tempfile.TemporaryDirectory() as d:
        for nm in suite_names():
            write_free_mps(load_golden_lp(nm), Path(d) / f"{nm}.mps")
        (Path(d) / "zz_broken.mps").write_text("NAME broken\nROWS\n N OBJ\nCOLUMNS\n X0 NOSUCHROW 1\nENDATA\n")
        run = text_call(L.ref_bench_run, d.encode(), C.byref(replace(p, time_limit_seconds=60.0).to_abi()),
                        60.0, 4)
    rows, aggs = [], []
    for line in run.splitlines()[2:]:
        f = line.split("\t")
        if f[0] == "aggregate":
            aggs.append({"group": f[1], "instances": int(f[2].split("=")[1]), "solved": int(f[3].split("=")[1])})
        else:
            rows.append({"instance": f[0], "nonzeros": int(f[1]), "status": f[2], "iterations": int(f[5]),
                         "primal_objective": float(f[6])})
    out["run"] = {"header": run.splitlines()[0], "columns": run.splitlines()[1], "rows": rows, "aggregates": aggs,
                  "eps_optimal": p.eps_optimal, "time_limit": 60.0}
    OUT.write_text(json.dumps(out, indent=1, default=lambda x: x) + "\n")
    print("wrote", OUT, len(rows), "instances")


if __name__ == "__main__":
    main()
