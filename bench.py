#!/usr/bin/env python3
"""Benchmark: restarted-PDHG iterations/s and time to 1e-4 relative KKT on
BASELINE.json configs[3] (C4: synthetic random sparse LP, m = 2e7 rows
(1e7 inequalities + 1e7 equalities), n = 4e7 columns, 5 nonzeros per column,
nnz = 2e8, fp64), the largest configuration one B200 holds. C2 (configs[1],
the 1k x 1k transportation LP, to 1e-4 and 1e-8) is reported beside it.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step is one complete solve of the device-resident instance from z = 0 to
1e-4 relative KKT (the reference's solve_seconds scope, solver.hpp:636-646,
760). `value` = PDHG iterations of all ranks / max-over-ranks device time of
the K timed solves (CUDA events on the solver's stream, inside libpdlp_b200).
`e2e` = the same metric through the C-ABI with host buffers: pdlp_create
(H2D of the 2.4 GB instance, K^T build, preconditioning, panel plans) +
pdlp_solve + pdlp_get_solution (D2H of x, y, lambda) every step. The inputs
(> 4 GB) exceed the 126 MB L2; L2 is also flushed between timed solves.
N > 1 (torchrun, one process per GPU, device = LOCAL_RANK): ONE row-sharded
solve of the instance (ShardRank: K and K^T cut by rows into N contiguous
ranges, each rank computing its rows of y' / Kx' and its columns of x' / K'y'
and pushing them into the peers' buffers inside the kernels, csrc/shard.cuh);
`value` = iterations of the instance / max-over-ranks device time ("scaling":
"strong"). --replicas runs N independent solves instead (weak scaling), which
is also the fallback, reported in `config.parallelism`, if the sharded setup
fails.

--impl reference times the reference CPU solver (oracle/_ref: the unmodified
pdhglp headers compiled in place) on the host cores: one shared setup of the
same C4 instance (SolveLoop's scaling and saddle form), then one concurrent
solve per core (forked iterate states), each step a bounded iteration sample;
rank 0 only. The reference cannot reach 1e-4 on C4 in bench time (about 5 s
per iteration on one core), so the metric there is iterations/s.
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
CONFIG = "C4"
WORKLOAD = ("C4 synthetic random sparse LP (BASELINE configs[3]): m=20,000,000 (10M inequality + 10M equality "
            "rows), n=40,000,000, nnz=200,000,000, boxes [0,10], fp64, z0=0 to 1e-4 relative KKT")
C2_WORKLOAD = "C2 synthetic transportation LP 1000 x 1000 (n=1,000,000, m=2,000, nnz=2,000,000)"
E2E_STEPS = 3


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


def profile_traffic(config: str):
    """Per-launch DRAM traffic (ncu dram__bytes_read + write) of the dual and
    primal kernel groups of `config` from the committed ncu summary."""
    p = ROOT / "profiles" / "ncu_summary.json"
    if p.exists():
        try:
            d = json.loads(p.read_text())
            return d.get(config, {})
        except Exception:
            return {}
    return {}


def mem_available_gb() -> float:
    try:
        for ln in open("/proc/meminfo"):
            if ln.startswith("MemAvailable:"):
                return float(ln.split()[1]) / 1048576.0
    except OSError:
        pass
    return 0.0


def reference_sessions(lp, threads: int):
    """One reference session (setup: make_scaling, apply_scaling, to_saddle)
    plus threads-1 forks sharing it. Falls back to the C port when the
    reference harness is not built."""
    from oracle import oracle as O
    from paper_2311_12180_b200 import SolverParams

    kind = "ref" if O.available("ref") else "oracle"
    t = time.perf_counter()
    s0 = O.Session(lp, SolverParams(iteration_limit=10**9, time_limit_seconds=1e9), kind)
    setup = time.perf_counter() - t
    sess = [s0]
    if kind == "ref":
        sess += [s0.fork() for _ in range(threads - 1)]
    return kind, sess, setup


def run_sessions(sess, iters: int) -> float:
    """Runs `iters` iterations on every session concurrently (ctypes drops the
    GIL); returns the aggregate iterations/s of the step."""
    ts = [threading.Thread(target=s.run, args=(iters,)) for s in sess]
    t = time.perf_counter()
    for th in ts:
        th.start()
    for th in ts:
        th.join()
    return len(sess) * iters / (time.perf_counter() - t)


def cpu_sample_main(args) -> None:
    """Child process of our arm: the reference on one host core, on a bounded
    sample of the bench workload (setup, then --cpu-iters iterations)."""
    from paper_2311_12180_b200 import generators

    try:
        os.sched_setaffinity(0, {max(os.sched_getaffinity(0))})
    except (AttributeError, OSError):
        pass
    lp = generators.config(CONFIG)
    kind, sess, setup = reference_sessions(lp, 1)
    sess[0].run(1)  # first iteration: page-in of the saddle operators
    rate = run_sessions(sess, args.cpu_iters)
    print(json.dumps({"value": rate, "unit": UNIT, "kind": "reference" if kind == "ref" else "port", "cores": 1,
                      "sample": f"{args.cpu_iters} iterations of the same {CONFIG} instance on 1 core after the "
                                f"reference's setup ({setup:.0f} s, outside the sample, as solve_seconds)"}),
          flush=True)


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return
    from paper_2311_12180_b200 import generators

    lp = generators.config(CONFIG)
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    # each forked solve holds ~5 (n + m) doubles of iterate state (C4: ~2.4 GB) plus
    # the step's temporaries; the shared setup ~16 B/nnz per matrix copy
    per = 8.0 * 10 * (lp.num_variables + lp.num_constraints) / 2**30
    shared = 8 * 16.0 * lp.nnz / 2**30
    threads = int(max(1, min(cores, 32, (mem_available_gb() - shared - 8.0) // max(per, 1e-3))))
    kind, sess, setup = reference_sessions(lp, threads)
    iters = max(1, args.ref_iters)
    for _ in range(args.warmup):
        run_sessions(sess, iters)
    vals = [run_sessions(sess, iters) for _ in range(args.steps)]
    for s in sess:
        s.close()
    value = float(np.mean(vals))
    desc = {"kind": "reference" if kind == "ref" else "port", "cores": threads,
            "sample": f"{iters} iteration(s) per step on each of {threads} concurrent solves of the same "
                      f"{CONFIG} instance (one shared reference setup of {setup:.0f} s, outside the timing, "
                      f"as solve_seconds; forked iterate states)"}
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generator)",
        "config": {"workload": WORKLOAD, "eps": 1e-4, "seed": generators.SEEDS[CONFIG]},
        "cpu_baseline": {"value": value, "unit": UNIT, **desc},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def c2_extra(device: int) -> dict:
    """C2 (BASELINE configs[1]) beside the headline: device-timed solves to
    1e-4 and 1e-8 (one warm solve each) and the iteration-kernel timings."""
    from paper_2311_12180_b200 import Solver, SolverParams, generators

    lp = generators.config("C2")
    out = {"workload": C2_WORKLOAD}
    for eps in (1e-4, 1e-8):
        with Solver(lp, SolverParams(eps_optimal=eps, device=device)) as s:
            s.solve()
            r = s.solve()
            out[f"solve_{eps:g}"] = {"status": str(r.status), "iterations": r.iterations,
                                     "device_ms": 1e3 * r.info["device_seconds"],
                                     "it_per_s": r.iterations / r.info["device_seconds"],
                                     "primal_objective": r.info["primal_objective"]}
            if eps == 1e-4:
                for which, name in ((0, "dual"), (1, "primal")):
                    ms, alg = s.time_kernel(which, 200)
                    kb = s.kernel_bytes(which)
                    out[f"{name}_us"] = 1e3 * ms
                    out[f"{name}_alg_gbs"] = alg / (ms * 1e-3) / 1e9
                    out[f"{name}_moved_gbs"] = kb["moved"] / (ms * 1e-3) / 1e9
    out["note"] = "working set ~130 MB: L2-resident across iterations (an L2/latency figure, not HBM)"
    return out


def run_ours(args):
    import torch

    rank, world, local = env_rank()
    dist = None
    device = 0
    if world > 1:
        import torch.distributed as dist

        ndev = max(1, torch.cuda.device_count())
        device = local % ndev
        torch.cuda.set_device(device)
        # several ranks per GPU (tests on a one-GPU box): NCCL refuses shared devices
        dist.init_process_group("nccl" if world <= ndev else "gloo")
    torch.cuda.set_device(device)
    from paper_2311_12180_b200 import ShardRank, Solver, SolverParams, generators

    # the CPU baseline runs beside the GPU timing in a child process pinned to
    # the last core (reference setup on C4 takes minutes of host time)
    cpu_proc = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu_proc = subprocess.Popen([sys.executable, str(ROOT / "bench.py"), "--cpu-sample",
                                     "--cpu-iters", str(args.cpu_iters)], stdout=subprocess.PIPE,
                                    stderr=subprocess.PIPE, text=True)
    t = time.perf_counter()
    lp = generators.config(args.config)
    gen_s = time.perf_counter() - t
    n, m, nnz = lp.num_variables, lp.num_constraints, lp.nnz
    params = SolverParams(eps_optimal=1e-4, device=device)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{device}")

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()

    def allmax(v: float) -> float:
        if not dist:
            return float(v)
        on = f"cuda:{device}" if dist.get_backend() == "nccl" else "cpu"
        t_ = torch.tensor([float(v)], dtype=torch.float64, device=on)
        dist.all_reduce(t_, op=dist.ReduceOp.MAX)
        return float(t_.item())

    # N > 1: one row-sharded solve of the instance over all ranks (
    # each rank one GPU, x' / y' pushed to peers inside the kernels); replicas
    # (one independent solve per GPU) only if the sharded setup fails
    sharded = world > 1 and not args.replicas
    fallback = None

    def make():
        return ShardRank(lp, params, device=device) if sharded else Solver(lp, params)

    t = time.perf_counter()
    solver, err = None, ""
    try:
        solver = make()
    except Exception as e:  # noqa: BLE001 - reported in the JSON line
        err = f"{type(e).__name__}: {e}"
    if sharded and allmax(1.0 if solver is None else 0.0) > 0.0:
        if solver is not None:
            solver.close()
        fallback = (err or "a peer rank failed")[:300]
        sharded = False
        solver = make()
    elif solver is None:
        raise RuntimeError(err)
    setup_s = time.perf_counter() - t
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
    max_dev_s = allmax(dev_s)
    # sharded: every rank runs the same iterations of the one instance; replicas: every rank its own
    total_iters = float(iters) if sharded or not dist else float(iters) * world
    value = total_iters / max_dev_s
    last = results[-1]

    # ---- roofline of the dominant kernel group (dual: K x' + update; primal: K'y' + update), one GPU ----
    peak, peak_kind = peaks()
    kern, dk, dom, traffic = {}, None, None, {}
    if world == 1:
        for which, name in ((0, "dual"), (1, "primal"), (2, "spmv_K"), (3, "spmv_KT")):
            ms, alg = solver.time_kernel(which, 20)
            kb = solver.kernel_bytes(which)
            kern[name] = {"us": 1e3 * ms, "alg_bytes": alg, "moved_bytes": kb["moved"], "panels": kb["panels"],
                          "alg_gbs": alg / (ms * 1e-3) / 1e9, "moved_gbs": kb["moved"] / (ms * 1e-3) / 1e9}
        dom = "primal" if kern["primal"]["us"] >= kern["dual"]["us"] else "dual"
        dk = kern[dom]
        traffic = profile_traffic(CONFIG).get(dom, {})
    solver.close()

    # the CPU baseline child ends before the end-to-end loop, whose host work
    # (uploads, setup) it would otherwise slow down
    cpu = None
    if cpu_proc is not None:
        out, err = cpu_proc.communicate(timeout=1800)
        try:
            cpu = json.loads(out.strip().splitlines()[-1])
        except (ValueError, IndexError):
            cpu = {"value": None, "unit": UNIT, "kind": "reference", "cores": 1,
                   "sample": f"failed: {err.strip()[-300:]}"}

    # ---- e2e through the C-ABI with host buffers ----
    e2e_steps = max(1, min(args.steps, E2E_STEPS))
    e2e_iters, e2e_s = 0, 0.0
    h2d = lp_bytes(lp)
    d2h = 8 * (2 * lp.num_variables + lp.num_constraints)  # x, y, lambda
    parts = {"create_ms": 0.0, "solve_ms": 0.0, "destroy_ms": 0.0}
    for _ in range(e2e_steps):
        flush.fill_(1.0)
        barrier()
        t0 = time.perf_counter()
        s2 = make()  # pdlp_create (+ the shard link): H2D + K^T + preconditioning + plans
        t1 = time.perf_counter()
        r2 = s2.solve()  # pdlp_solve + pdlp_get_solution (D2H)
        t2 = time.perf_counter()
        s2.close()  # pdlp_destroy
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        e2e_s += t3 - t0
        parts["create_ms"] += 1e3 * (t1 - t0) / e2e_steps
        parts["solve_ms"] += 1e3 * (t2 - t1) / e2e_steps
        parts["destroy_ms"] += 1e3 * (t3 - t2) / e2e_steps
        e2e_iters += r2.iterations
    e2e_total = float(e2e_iters) if sharded or not dist else float(e2e_iters) * world
    e2e_value = e2e_total / allmax(e2e_s)
    del lp

    c2 = c2_extra(device) if rank == 0 and world == 1 and not args.no_c2 else None


    if rank == 0:
        if world == 1:
            par = "single GPU"
        elif sharded:
            par = f"row-sharded x{world} (one instance; x', y' pushed to peers inside the kernels, csrc/shard.cuh)"
        else:
            par = f"replicas x{world}" + (f" (sharded setup failed: {fallback})" if fallback else "")
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * max_dev_s / args.steps, "higher_is_better": True,
            "scaling": "strong" if sharded else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generator, no dataset)",
            "config": {"workload": WORKLOAD if args.config == CONFIG else args.config, "eps": 1e-4,
                       "seed": generators.SEEDS[args.config], "parallelism": par,
                       "l2": "inputs (>4 GB) exceed L2; also flushed between timed solves (256 MiB write)"},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d * (world if sharded else 1),
                    "d2h_bytes_per_step": d2h * (world if sharded else 1), "steps": e2e_steps, "per_step": parts},
            "time_to_tolerance_ms": 1e3 * last.info["device_seconds"], "iterations": last.iterations,
            "window_ms": 1e3 * last.info["window_seconds"], "eval_ms": 1e3 * last.info["eval_seconds"],
            "windows_chained": last.info["eval_seconds"] == 0.0,
            "host_gap_ms": 1e3 * (last.info["device_seconds"] - last.info["window_seconds"]
                                  - last.info["eval_seconds"]),
            "restarts": last.restarts, "status": str(last.status),
            "primal_objective": last.info["primal_objective"],
            "setup_ms": 1e3 * last.info["setup_seconds"], "create_s": setup_s, "generate_s": gen_s,
            "gpu_launches": int(launches), "clocks": clk, "wall_s": wall,
        }
        if dk is not None:
            line["roofline"] = {"bound": "hbm", "kernel": dom, "achieved": dk["alg_gbs"], "peak": peak, "unit": "GB/s",
                                "frac": dk["alg_gbs"] / peak, "traffic": traffic.get("dram_bytes_per_launch"),
                                "peak_source": peak_kind, "bytes_per_launch": dk["alg_bytes"],
                                "moved_bytes_per_launch": dk["moved_bytes"], "moved_frac": dk["moved_gbs"] / peak,
                                "launch_us": dk["us"], "panels": dk["panels"],
                                "traffic_source": traffic.get("source")}
            line["iteration_roofline"] = {"b_iter_bytes": b_iter(n, m, nnz),
                                          "achieved_gbs": b_iter(n, m, nnz) * value / 1e9,
                                          "frac": b_iter(n, m, nnz) * value / 1e9 / peak}
            line["kernels"] = kern
        else:
            line["iteration_roofline"] = {"b_iter_bytes": b_iter(n, m, nnz),
                                          "achieved_gbs_per_gpu": b_iter(n, m, nnz) * value / world / 1e9,
                                          "frac_per_gpu": b_iter(n, m, nnz) * value / world / 1e9 / peak}
        if c2:
            line["c2"] = c2
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
    ap.add_argument("--cpu-iters", type=int, default=4, help="CPU baseline sample (iterations, 1 core)")
    ap.add_argument("--ref-iters", type=int, default=1, help="reference arm: iterations per solve per step")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-c2", action="store_true")
    ap.add_argument("--replicas", action="store_true", help="N > 1: independent replicas instead of one sharded solve")
    ap.add_argument("--config", default=CONFIG, help=argparse.SUPPRESS)  # tests: a smaller config
    ap.add_argument("--cpu-sample", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.cpu_sample:
        cpu_sample_main(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
