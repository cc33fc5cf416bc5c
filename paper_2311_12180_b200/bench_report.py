"""Benchmark report over a directory of MPS instances, solved on the B200.

Host-side mirror of the reference's benchmark harness (pdhglp/bench.hpp) with
the same names, numbers and file format, so reports from the two solvers can
be diffed line by line:

* shifted_geometric_mean  bench.hpp:29-41  (SGM10 is shift = 10)
* size_class_for          bench.hpp:56-60  ([0, 1M) small, [1M, 10M) medium, else large)
* BenchmarkRecord         bench.hpp:62-82
* aggregate_records       bench.hpp:109-130 (time limit for inconclusive runs,
                                             parse failures excluded)
* config_hash             bench.hpp:135-155 (FNV-1a over the canonical parameter string)
* solve_instance_for_benchmark  bench.hpp:157-183 (read_mps + the GPU solve)
* run_benchmark           bench.hpp:190-238 (sorted *.mps / *.mps.gz, `jobs` workers)
* write_report            bench.hpp:242-262 (header, tab-separated rows, aggregates)

The solves go through the GPU library; only the bookkeeping is Python. Worker
threads each own their solver handle (one handle per host thread, the C-ABI's
rule); with several visible GPUs, worker w uses device w % device_count.
"""
from __future__ import annotations

import enum
import math
import os
import threading
import time
from dataclasses import dataclass, field, replace
from pathlib import Path
from typing import Iterable, Sequence

from .lp import SolverParams, SolveStatus


def shifted_geometric_mean(times: Sequence[float], shift: float) -> float:
    """(prod_i (t_i + shift))^(1/n) - shift in log space (bench.hpp:29-41)."""
    if len(times) == 0:
        raise ValueError("shifted_geometric_mean: empty time list")
    log_sum = 0.0
    for t in times:
        if t < 0.0:
            raise ValueError("shifted_geometric_mean: negative time")
        log_sum += math.log(t + shift)
    return math.exp(log_sum / float(len(times))) - shift


class SizeClass(enum.IntEnum):
    SMALL = 0
    MEDIUM = 1
    LARGE = 2

    def __str__(self) -> str:  # to_string(SizeClass), bench.hpp:45-52
        return ("small", "medium", "large")[int(self)]


def size_class_for(nonzeros: int) -> SizeClass:
    """Inclusive lower thresholds; exactly 1,000,000 nonzeros is medium."""
    if nonzeros < 1_000_000:
        return SizeClass.SMALL
    if nonzeros < 10_000_000:
        return SizeClass.MEDIUM
    return SizeClass.LARGE


@dataclass
class BenchmarkRecord:
    instance: str
    nonzeros: int = 0
    parse_failed: bool = False
    parse_error: str = ""
    status: SolveStatus = SolveStatus.NUMERICAL_ERROR
    solve_seconds: float = 0.0  # scaling + solve, excludes parsing
    total_seconds: float = 0.0  # parse + scaling + solve
    iterations: int = 0
    primal_objective: float = 0.0
    relative_gap: float = 0.0
    relative_primal_residual: float = 0.0
    relative_dual_residual: float = 0.0

    def solved(self) -> bool:
        return not self.parse_failed and self.status in (
            SolveStatus.OPTIMAL, SolveStatus.PRIMAL_INFEASIBLE, SolveStatus.DUAL_INFEASIBLE)


@dataclass
class AggregateRow:
    group: str
    instances: int = 0
    solved: int = 0
    sgm10: float = 0.0


@dataclass
class BenchmarkReport:
    config_line: str
    time_limit: float
    records: list[BenchmarkRecord] = field(default_factory=list)
    aggregates: list[AggregateRow] = field(default_factory=list)


def aggregation_time(r: BenchmarkRecord, time_limit: float) -> float:
    return min(r.solve_seconds, time_limit) if r.solved() else time_limit


def aggregate_records(records: Iterable[BenchmarkRecord], time_limit: float,
                      shift: float = 10.0) -> list[AggregateRow]:
    records = list(records)
    rows = []

    def build(group: str, keep) -> None:
        row = AggregateRow(group)
        times = []
        for r in records:
            if r.parse_failed or not keep(r):
                continue
            row.instances += 1
            row.solved += 1 if r.solved() else 0
            times.append(aggregation_time(r, time_limit))
        row.sgm10 = shifted_geometric_mean(times, shift) if times else 0.0
        rows.append(row)

    for c in SizeClass:
        build(str(c), lambda r, c=c: size_class_for(r.nonzeros) == c)
    build("total", lambda r: True)
    return rows


def _g(x: float, digits: int) -> str:
    """std::ostream << double with precision(digits) (the %g style)."""
    if math.isnan(x):
        return "-nan" if math.copysign(1.0, x) < 0 else "nan"
    return f"{x:.{digits}g}"


def config_hash(p: SolverParams, time_limit: float) -> str:
    """FNV-1a 64 over the canonical parameter string (bench.hpp:135-155)."""
    parts = [
        _g(p.eps_optimal, 17), _g(p.eps_infeasible, 17), _g(time_limit, 17), str(int(p.iteration_limit)),
        _g(p.beta_sufficient, 17), _g(p.beta_necessary, 17), _g(p.beta_artificial, 17),
        _g(p.theta_smoothing, 17), _g(p.eps_zero, 17), str(int(p.evaluation_frequency)), str(int(p.scaling)),
        str(int(p.ruiz_iterations)), _g(p.pock_chambolle_alpha, 17), _g(p.step_reduction_exponent, 17),
        _g(p.step_growth_exponent, 17), _g(p.omega_min, 17), _g(p.omega_max, 17),
    ]
    h = 14695981039346656037
    for ch in "|".join(parts).encode():
        h ^= ch
        h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"


def solve_instance_for_benchmark(path: str | os.PathLike, params: SolverParams) -> BenchmarkRecord:
    """read_mps + solve on the GPU, timed like bench.hpp:157-183."""
    from .api import read_mps, solve

    rec = BenchmarkRecord(instance=Path(path).name)
    t0 = time.perf_counter()
    try:
        lp = read_mps(path)
    except (ValueError, RuntimeError, OSError) as e:  # MpsParseError / runtime_error
        rec.parse_failed = True
        rec.parse_error = str(e)
        return rec
    rec.nonzeros = lp.nnz
    r = solve(lp, params)
    rec.status = r.status
    rec.solve_seconds = min(r.solve_seconds, params.time_limit_seconds)  # the record invariant
    rec.total_seconds = time.perf_counter() - t0
    rec.iterations = r.iterations
    rec.primal_objective = r.info["primal_objective"]
    rec.relative_gap = r.info["relative_gap"]
    rec.relative_primal_residual = r.info["relative_primal_residual"]
    rec.relative_dual_residual = r.info["relative_dual_residual"]
    return rec


def run_benchmark(directory: str | os.PathLike, params: SolverParams, time_limit: float,
                  jobs: int = 1) -> BenchmarkReport:
    """Every *.mps / *.mps.gz directly under `directory`, records ordered by
    instance name; unsolved runs count the time limit, parse failures are
    listed but excluded from the aggregates (bench.hpp:190-238)."""
    params = replace(params, time_limit_seconds=time_limit)
    paths = sorted(str(e) for e in Path(directory).iterdir()
                   if e.is_file() and (e.name.endswith(".mps") or e.name.endswith(".mps.gz")))
    records: list[BenchmarkRecord | None] = [None] * len(paths)
    if jobs <= 1:
        for i, p in enumerate(paths):
            records[i] = solve_instance_for_benchmark(p, params)
    else:
        from .api import device_count

        ndev = max(1, device_count())
        lock = threading.Lock()
        nxt = [0]
        errors: list[BaseException] = []

        def worker(w: int) -> None:
            wp = replace(params, device=(params.device + w) % ndev)
            while True:
                with lock:
                    i = nxt[0]
                    nxt[0] += 1
                if i >= len(paths):
                    return
                try:
                    records[i] = solve_instance_for_benchmark(paths[i], wp)
                except BaseException as e:  # surfaced after the join
                    errors.append(e)
                    return

        threads = [threading.Thread(target=worker, args=(w,)) for w in range(min(jobs, len(paths)))]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        if errors:
            raise errors[0]
    recs = sorted((r for r in records if r is not None), key=lambda r: r.instance)
    return BenchmarkReport(config_hash(params, time_limit), time_limit, recs,
                           aggregate_records(recs, time_limit))


def report_text(report: BenchmarkReport) -> str:
    """The report file's contents (bench.hpp:242-262): doubles at precision 9."""
    out = [f"# pdhglp benchmark report config={report.config_line} time_limit={_g(report.time_limit, 9)}\n",
           "instance\tnonzeros\tstatus\tsolve_seconds\ttotal_seconds\titerations"
           "\tprimal_objective\trelative_gap\trelative_primal_residual\trelative_dual_residual\n"]
    for r in report.records:
        if r.parse_failed:
            out.append(f"{r.instance}\t0\tparse_error\t0\t0\t0\t0\t0\t0\t0\n")
            continue
        out.append("\t".join([r.instance, str(r.nonzeros), str(SolveStatus(r.status)), _g(r.solve_seconds, 9),
                              _g(r.total_seconds, 9), str(r.iterations), _g(r.primal_objective, 9),
                              _g(r.relative_gap, 9), _g(r.relative_primal_residual, 9),
                              _g(r.relative_dual_residual, 9)]) + "\n")
    for a in report.aggregates:
        out.append(f"aggregate\t{a.group}\tinstances={a.instances}\tsolved={a.solved}\tsgm10={_g(a.sgm10, 9)}\n")
    return "".join(out)


def write_report(report: BenchmarkReport, path: str | os.PathLike) -> None:
    try:
        with open(path, "w") as f:
            f.write(report_text(report))
    except OSError as e:
        raise RuntimeError(f"cannot write '{path}'") from e
