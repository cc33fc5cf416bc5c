"""The directory benchmark (bench_report.run_benchmark and the C++ header's
run_benchmark) on the B200 against the reference's own run_benchmark over the
same files (tests/golden/bench_golden.json, make_golden_bench.py): the 25
golden instances written back as MPS plus one unparsable file.

Bars: the same header (config hash, time limit) and column line; per instance
the same nonzeros and status, objective within the solve tolerance; the parse
failure listed with zeros and left out of the aggregates; the same aggregate
instance / solved counts."""
from __future__ import annotations

import json
import subprocess
from pathlib import Path

import pytest

from paper_2311_12180_b200 import SolverParams
from paper_2311_12180_b200 import bench_report as B
from tests.helpers import load_golden_lp, suite_names, write_free_mps

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
GOLD = json.loads((ROOT / "tests" / "golden" / "bench_golden.json").read_text())["run"]


@pytest.fixture(scope="module")
def mps_dir(tmp_path_factory) -> Path:
    d = tmp_path_factory.mktemp("suite_mps")
    for nm in suite_names():
        write_free_mps(load_golden_lp(nm), d / f"{nm}.mps")
    (d / "zz_broken.mps").write_text("NAME broken\nROWS\n N OBJ\nCOLUMNS\n X0 NOSUCHROW 1\nENDATA\n")
    (d / "notes.txt").write_text("not an instance\n")
    return d


def check_report(text: str) -> None:
    lines = text.splitlines()
    assert lines[0] == GOLD["header"] and lines[1] == GOLD["columns"]
    rows = [ln.split("\t") for ln in lines[2:] if not ln.startswith("aggregate")]
    aggs = [ln.split("\t") for ln in lines[2:] if ln.startswith("aggregate")]
    assert [r[0] for r in rows] == [g["instance"] for g in GOLD["rows"]]
    for r, g in zip(rows, GOLD["rows"]):
        assert int(r[1]) == g["nonzeros"] and r[2] == g["status"], (r, g)
        if g["status"] == "optimal":
            obj = float(r[6])
            assert abs(obj - g["primal_objective"]) <= 1e-3 * (1.0 + abs(g["primal_objective"])), (r, g)
        if g["status"] == "parse_error":
            assert r[1:] == ["0", "parse_error"] + ["0"] * 7
    assert [(a[1], int(a[2].split("=")[1]), int(a[3].split("=")[1])) for a in aggs] == \
        [(g["group"], g["instances"], g["solved"]) for g in GOLD["aggregates"]]


@pytest.mark.parametrize("jobs", [1, 3])
def test_python_run_benchmark_matches_reference_report(mps_dir, jobs, tmp_path):
    rep = B.run_benchmark(mps_dir, SolverParams(eps_optimal=GOLD["eps_optimal"]), GOLD["time_limit"], jobs=jobs)
    out = tmp_path / "report.tsv"
    B.write_report(rep, out)
    check_report(out.read_text())
    assert all(r.solve_seconds <= GOLD["time_limit"] for r in rep.records)
    assert [r.instance for r in rep.records] == sorted(r.instance for r in rep.records)


def test_cpp_header_run_benchmark_matches_reference_report(mps_dir, tmp_path):
    exe = tmp_path / "brp"
    lib = ROOT / "paper_2311_12180_b200" / "lib"
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", str(ROOT / "include"),
                    str(ROOT / "tests" / "cpp" / "bench_report_probe.cpp"), "-o", str(exe), f"-L{lib}",
                    "-lpdlp_b200", f"-Wl,-rpath,{lib}"], check=True)
    out = subprocess.run([str(exe), "dir", str(mps_dir), repr(GOLD["time_limit"]), "2"], capture_output=True,
                         text=True, check=True, timeout=600).stdout
    check_report(out)
