#!/usr/bin/env python3
"""Benchmark: restarted-PDHG iterations/s on BASELINE.json configs[1] (C2:
synthetic 1000 x 1000 transportation LP, n = 1e6, m = 2000, nnz = 2e6, solved
from z = 0 to 1e-4 relative KKT).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step is one complete solve on the device-resident instance (the reference's
solve_seconds scope, solver.hpp:636-646,760). `value` = total PDHG iterations of
all ranks / max-over-ranks device time of the K timed solves (CUDA events on the
solver's stream, inside libpdlp_b200). `e2e` = the same metric through the
C-ABI with host buffers: pdlp_create (H2D, K^T build, preconditioning) +
pdlp_solve + pdlp_get_solution (D2H) every step. C2 fits one GPU many times
over and does not shard ("C1 and C2 ... run them as replicas
only"), so N > 1 runs N independent replicas (weak scaling, no collective on the
data path). L2 (126 MB) is flushed between timed solves with a 256 MiB write.

--impl reference times the reference CPU solver (oracle/_ref, the unmodified
pdhglp headers compiled in place) on the host cores: one solve per core, each a
bounded iteration sample of the same instance; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "PDHG iters/sec (solve to 1e-4 relative KKT)"
UNIT = "iter/s"
WORKLOAD = "C2 synthetic transportation LP 1000 sources x 1000 sinks (n=1,000,000, m=2,000, nnz=2,000,000), fp64, z0=0 to 1e-4 relative KKT"
CPU_SAMPLE_ITERS = 384


def env_rank():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


def peaks():
    """HBM peak for the roofline: MEASURED_PEAKS.json (driver-written) when
    present -- its burst figure, since the dominant kernel is timed alone --
    else the 6650 GB/s fallback of B200_PROFILING.md."""
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            d = json.loads(p.read_text())
        except ValueError:
            d = {}
        flat = {}

        def walk(o, pre=""):
            if isinstance(o, dict):
                for k, v in o.items():
                    walk(v, f"{pre}{k}.".lower())
            elif isinstance(o, (int, float)) and not isinstance(o, bool):
                flat[pre.rstrip(".")] = float(o)

        walk(d)
        hbm = {k: v for k, v in flat.items() if "hbm" in k and v > 100.0}
        for pref in ("burst", "hbm_gbs", "copy", "sustained", ""):
            cand = [v for k, v in sorted(hbm.items()) if pref in k]
            if cand:
                return cand[0], "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled DURING the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.proc, self.lines = index, None, []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def b_iter(n: int, m: int, nnz: int) -> float:
    """Algorithmic bytes per accepted single-trial iteration."""
    return 24.0 * nnz + 4.0 * (m + n + 2) + 8.0 * (10 * n + 8 * m)


def lp_bytes(lp) -> int:
    tot = 0
    for M in (lp.inequality_matrix, lp.equality_matrix):
        tot += M.row_offsets.nbytes + M.col_indices.nbytes + M.values.nbytes
    for v in (lp.objective, lp.inequality_rhs, lp.equality_rhs, lp.lower, lp.upper):
        tot += v.nbytes
    return tot


def profile_traffic():
    """Per-launch DRAM traffic of the primal kernel from the committed ncu summary."""
    p = ROOT / "profiles" / "ncu_summary.json"
    if p.exists():
        try:
            d = json.loads(p.read_text())
            return d.get("primal_kernel", {}).get("dram_bytes_per_launch")
        except Exception:
            return None
    return None


def cpu_reference_rate(lp, iters: int, threads: int) -> tuple[float, dict]:
    """The reference solver (oracle/_ref) on `threads` host cores, one
    independent bounded solve per core; aggregate = sum of per-core rates."""
    from oracle import oracle as O
    from paper_2311_12180_b200 import SolverParams

    kind = "ref" if O.available("ref") else "oracle"
    params = SolverParams(iteration_limit=iters, time_limit_seconds=600.0)
    rates = [0.0] * threads

    def work(i):
        r = O.solve(lp, params, kind)
        rates[i] = r.iterations / max(r.solve_seconds, 1e-12)

    ts = [threading.Thread(target=work, args=(i,)) for i in range(threads)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    return float(sum(rates)), {"kind": "reference" if kind == "ref" else "port", "cores": threads,
                               "sample": f"{iters} iterations of the same C2 instance per core after setup "
                                         f"(the reference's solve_seconds scope), {threads} concurrent solve(s)"}


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return
    from paper_2311_12180_b200 import generators

    lp = generators.config("C2")
    threads = max(1, min(os.cpu_count() or 1, 32))
    for _ in range(args.warmup):
        cpu_reference_rate(lp, 16, threads)
    vals = []
    desc = None
    for _ in range(args.steps):
        v, desc = cpu_reference_rate(lp, args.cpu_iters, threads)
        vals.append(v)
    value = float(np.mean(vals))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generator)",
        "config": {"workload": WORKLOAD, "eps": 1e-4, "seed": generators.SEEDS["C2"]},
        "cpu_baseline": {"value": value, "unit": UNIT, **desc},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch

    rank, world, local = env_rank()
    dist = None
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    device = local if world > 1 else 0
    torch.cuda.set_device(device)
    from paper_2311_12180_b200 import Solver, SolverParams, SolveStatus, generators

    lp = generators.config("C2")
    params = SolverParams(eps_optimal=1e-4, device=device)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{device}")

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()

    solver = Solver(lp, params)
    for _ in range(args.warmup):
        solver.solve()
    # ---- timed region (device-resident inputs) ----
    clocks = ClockSampler(device)
    barrier()
    clocks.start()
    iters = 0
    dev_s = 0.0
    wall0 = time.perf_counter()
    launches = 0
    results = []
    for _ in range(args.steps):
        flush.fill_(1.0)  # evict the 126 MB L2 between solves
        torch.cuda.synchronize()
        r = solver.solve()
        iters += r.iterations
        dev_s += r.info["device_seconds"]
        launches += r.info["gpu_launches"]
        results.append(r)
    barrier()
    wall = time.perf_counter() - wall0
    clk = clocks.stop()
    t = torch.tensor([dev_s], dtype=torch.float64, device=f"cuda:{device}")
    it_t = torch.tensor([float(iters)], dtype=torch.float64, device=f"cuda:{device}")
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(it_t, op=dist.ReduceOp.SUM)
    max_dev_s, total_iters = float(t.item()), float(it_t.item())
    value = total_iters / max_dev_s
    last = results[-1]

    # ---- roofline of the dominant kernel (primal: K'y' fused update) ----
    peak, peak_kind = peaks()
    prim_ms, prim_bytes = solver.time_kernel(1, 200)
    dual_ms, dual_bytes = solver.time_kernel(0, 200)
    # time to 1e-8 relative KKT (BASELINE configs[1] quotes both tolerances), one solve
    with Solver(lp, SolverParams(eps_optimal=1e-8, device=device)) as s8:
        r8 = s8.solve()
    tol8 = {"status": str(r8.status), "iterations": r8.iterations, "device_ms": 1e3 * r8.info["device_seconds"],
            "primal_objective": r8.info["primal_objective"]}
    # plain SpMV over K and the stored K^T (BASELINE metric: "SpMV GB/s vs HBM peak")
    spmv = {}
    for which, name in ((2, "K"), (3, "KT")):
        ms_, by_ = solver.time_kernel(which, 200)
        spmv[name] = {"us": 1e3 * ms_, "bytes": by_, "gbs": by_ / (ms_ * 1e-3) / 1e9,
                      "frac": by_ / (ms_ * 1e-3) / 1e9 / peaks()[0]}
    solver.close()
    dom = "primal" if prim_ms >= dual_ms else "dual"
    ms, by = (prim_ms, prim_bytes) if dom == "primal" else (dual_ms, dual_bytes)
    achieved = by / (ms * 1e-3) / 1e9

    # ---- e2e through the C-ABI with host buffers ----
    e2e_iters, e2e_s = 0, 0.0
    h2d = lp_bytes(lp)
    d2h = 8 * (2 * lp.num_variables + lp.num_constraints)  # x, y, lambda
    parts = {"create_ms": 0.0, "solve_ms": 0.0, "destroy_ms": 0.0}
    for _ in range(max(1, args.steps)):
        flush.fill_(1.0)
        barrier()
        t0 = time.perf_counter()
        s2 = Solver(lp, params)  # pdlp_create: H2D + K^T + preconditioning
        t1 = time.perf_counter()
        r2 = s2.solve()  # pdlp_solve + pdlp_get_solution (D2H)
        t2 = time.perf_counter()
        s2.close()
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        e2e_s += t3 - t0
        parts["create_ms"] += 1e3 * (t1 - t0) / args.steps
        parts["solve_ms"] += 1e3 * (t2 - t1) / args.steps
        parts["destroy_ms"] += 1e3 * (t3 - t2) / args.steps
        e2e_iters += r2.iterations
    et = torch.tensor([e2e_s], dtype=torch.float64, device=f"cuda:{device}")
    ei = torch.tensor([float(e2e_iters)], dtype=torch.float64, device=f"cuda:{device}")
    if dist:
        dist.all_reduce(et, op=dist.ReduceOp.MAX)
        dist.all_reduce(ei, op=dist.ReduceOp.SUM)
    e2e_value = float(ei.item()) / float(et.item())

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        v, desc = cpu_reference_rate(lp, args.cpu_iters, 1)
        cpu = {"value": v, "unit": UNIT, **desc}

    if rank == 0:
        n, m, nnz = lp.num_variables, lp.num_constraints, lp.nnz
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * max_dev_s / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generator, no dataset)",
            "config": {"workload": WORKLOAD, "eps": 1e-4, "seed": generators.SEEDS["C2"],
                       "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
                       "l2": "flushed between timed solves (256 MiB write); working set ~130 MB"},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "per_step": parts},
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": profile_traffic(), "peak_source": peak_kind,
                         "bytes_per_launch": by, "launch_us": 1e3 * ms},
            "iteration_roofline": {"b_iter_bytes": b_iter(n, m, nnz),
                                   "achieved_gbs": b_iter(n, m, nnz) * value / world / 1e9,
                                   "frac": b_iter(n, m, nnz) * value / world / 1e9 / peak},
            "kernels_us": {"dual": 1e3 * dual_ms, "primal": 1e3 * prim_ms},
            "spmv": spmv,
            "solve_1e-8": tol8,
            "time_to_tolerance_ms": 1e3 * last.info["device_seconds"], "iterations": last.iterations,
            # with chained windows (the default graph engine) the evaluations run
            # inside the window graphs: window_ms then includes them
            "window_ms": 1e3 * last.info["window_seconds"], "eval_ms": 1e3 * last.info["eval_seconds"],
            "windows_chained": last.info["eval_seconds"] == 0.0,
            "host_gap_ms": 1e3 * (last.info["device_seconds"] - last.info["window_seconds"]
                                  - last.info["eval_seconds"]),
            "restarts": last.restarts, "status": str(last.status),
            "primal_objective": last.info["primal_objective"],
            "setup_ms": 1e3 * last.info["setup_seconds"],
            "gpu_launches": int(launches), "clocks": clk,
            "wall_s": wall,
        }
        if cpu:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-iters", type=int, default=CPU_SAMPLE_ITERS)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
