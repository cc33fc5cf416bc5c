"""The benchmark harness mirror (bench_report.py, include/pdlp_b200_bench.hpp)
against the reference's bench.hpp, through golden values the reference
produced (tests/golden/make_golden_bench.py): config hashes, SGM10 values and
the exact report text. CPU only: no solves here (test_gpu_bench_report.py runs
the directory benchmark on the B200)."""
from __future__ import annotations

import json
import math
import subprocess
from pathlib import Path

import pytest

from paper_2311_12180_b200 import SolverParams
from paper_2311_12180_b200 import bench_report as B
from paper_2311_12180_b200.lp import ScalingMode, SolveStatus

ROOT = Path(__file__).resolve().parents[1]
GOLD = json.loads((ROOT / "tests" / "golden" / "bench_golden.json").read_text())

PARAM_SETS = {  # tests/golden/make_golden_bench.py
    "default": SolverParams(),
    "eps8": SolverParams(eps_optimal=1e-8),
    "limit1000": SolverParams(iteration_limit=1000),
    "no_scaling": SolverParams(scaling=ScalingMode.NONE),
    "theta03_omega1e6": SolverParams(theta_smoothing=0.3, omega_max=1e6),
    "freq32_ruiz5": SolverParams(evaluation_frequency=32, ruiz_iterations=5, pock_chambolle_alpha=0.5),
}


def records_from_golden() -> list[B.BenchmarkRecord]:
    return [B.BenchmarkRecord(instance=r[0], nonzeros=r[1], parse_failed=bool(r[2]), status=SolveStatus(r[3]),
                              solve_seconds=r[4], total_seconds=r[5], iterations=r[6], primal_objective=r[7],
                              relative_gap=r[8], relative_primal_residual=r[9], relative_dual_residual=r[10])
            for r in GOLD["records"]]


def test_config_hash_matches_reference():
    for h in GOLD["hashes"]:
        assert B.config_hash(PARAM_SETS[h["params"]], h["time_limit"]) == h["hash"], h


def test_shifted_geometric_mean_matches_reference():
    for c in GOLD["sgm"]:
        v = B.shifted_geometric_mean(c["times"], c["shift"])
        assert v == pytest.approx(c["value"], rel=1e-15, abs=1e-15)
    with pytest.raises(ValueError, match="empty"):
        B.shifted_geometric_mean([], 10.0)
    with pytest.raises(ValueError, match="negative"):
        B.shifted_geometric_mean([1.0, -1e-9], 10.0)


def test_size_classes_inclusive_lower_thresholds():
    assert [str(B.size_class_for(v)) for v in (0, 999_999, 1_000_000, 9_999_999, 10_000_000)] == \
        ["small", "small", "medium", "medium", "large"]


def test_report_text_matches_reference_exactly():
    recs = records_from_golden()
    rep = B.BenchmarkReport(B.config_hash(SolverParams(), 60.0), 60.0, recs, B.aggregate_records(recs, 60.0))
    assert B.report_text(rep) == GOLD["report"]


def test_aggregation_rules():
    recs = records_from_golden()
    rows = {a.group: a for a in B.aggregate_records(recs, 60.0)}
    # parse failures excluded; the time limit stands in for inconclusive runs
    assert rows["total"].instances == len(recs) - 1
    assert rows["total"].solved == sum(r.solved() for r in recs)
    assert rows["medium"].instances == 2 and rows["large"].instances == 1  # 1,000,000 and 9,999,999 nnz
    small = [min(r.solve_seconds, 60.0) if r.solved() else 60.0
             for r in recs if not r.parse_failed and r.nonzeros < 1_000_000]
    assert rows["small"].sgm10 == pytest.approx(
        math.exp(sum(math.log(t + 10.0) for t in small) / len(small)) - 10.0, rel=1e-15)


def test_write_report_error_is_runtime_error(tmp_path):
    rep = B.BenchmarkReport("x", 1.0)
    with pytest.raises(RuntimeError, match="cannot write"):
        B.write_report(rep, tmp_path / "no" / "such" / "dir" / "r.tsv")


@pytest.fixture(scope="module")
def probe(tmp_path_factory) -> Path:
    """tests/cpp/bench_report_probe.cpp against the C++ header."""
    d = tmp_path_factory.mktemp("probe")
    exe = d / "brp"
    lib = ROOT / "paper_2311_12180_b200" / "lib"
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", str(ROOT / "include"),
                    str(ROOT / "tests" / "cpp" / "bench_report_probe.cpp"), "-o", str(exe), f"-L{lib}",
                    "-lpdlp_b200", f"-Wl,-rpath,{lib}"], check=True)
    return exe


def test_cpp_header_config_hash_matches_reference(probe):
    for h in GOLD["hashes"]:
        p = PARAM_SETS[h["params"]]
        args = [repr(p.eps_optimal), str(p.iteration_limit), str(int(p.scaling)), repr(p.theta_smoothing),
                repr(p.omega_max), str(p.evaluation_frequency), str(p.ruiz_iterations),
                repr(p.pock_chambolle_alpha), repr(h["time_limit"])]
        out = subprocess.run([str(probe), "hash", *args], capture_output=True, text=True, check=True).stdout
        assert out.strip() == h["hash"], h


def test_cpp_header_report_matches_reference(probe, tmp_path):
    tsv = tmp_path / "records.tsv"
    tsv.write_text("".join(" ".join(repr(v) if isinstance(v, float) else str(v) for v in r) + "\n"
                           for r in GOLD["records"]))
    out = subprocess.run([str(probe), "report", str(tsv), "60"], capture_output=True, text=True, check=True).stdout
    assert out == GOLD["report"]


def test_acceptance_criterion_8_hand_values():
    """acceptance_main.cpp:505-520: SGM10 of [10, 90] and the time-limit
    contribution of an inconclusive record."""
    assert abs(B.shifted_geometric_mean([10.0, 90.0], 10.0) - 34.7214) <= 1e-3
    unsolved = B.BenchmarkRecord(instance="u", status=SolveStatus.TIME_LIMIT, solve_seconds=123.0)
    assert B.aggregation_time(unsolved, 77.0) == 77.0
