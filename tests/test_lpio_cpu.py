"""CPU tests of the host-side LP I/O in libpdlp_b200.so (no GPU): the MPS
reader against the REFERENCE reader (mps_io.hpp, via oracle/_ref) on every
fixture the reference ships, the golden instances, error lines of the bad
fixtures, the solution file, and the C++ host header compiled against the
library."""
from __future__ import annotations

import glob
import os
import subprocess
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle as O
from paper_2311_12180_b200 import CsrMatrix, GeneralFormLp, PdlpError, parse_mps, read_mps, write_solution
from paper_2311_12180_b200.api import MPS_FIXED, MPS_FREE, library_path
from tests.helpers import lp_hash, ref_suite

ROOT = Path(__file__).resolve().parents[1]
FIX = Path("/root/reference/proj/tests/fixtures")
needs_fixtures = pytest.mark.skipif(not FIX.exists() or not O.available("ref"),
                                    reason="reference fixtures / oracle/_ref not present")


def fixtures() -> list[str]:
    if not FIX.exists():
        return []
    return sorted(glob.glob(str(FIX / "*.mps")) + glob.glob(str(FIX / "suite" / "*.mps")))


def same_lp(a: GeneralFormLp, b: GeneralFormLp) -> bool:
    for x, y in ((a.inequality_matrix, b.inequality_matrix), (a.equality_matrix, b.equality_matrix)):
        if not (x.num_rows == y.num_rows and np.array_equal(x.row_offsets, y.row_offsets)
                and np.array_equal(x.col_indices.astype(np.int64), y.col_indices.astype(np.int64))
                and np.array_equal(x.values, y.values)):
            return False
    return all(np.array_equal(getattr(a, k), getattr(b, k)) for k in
               ("objective", "inequality_rhs", "equality_rhs", "lower", "upper")) and \
        np.signbit(a.objective_constant) == np.signbit(b.objective_constant) and \
        a.objective_constant == b.objective_constant


@needs_fixtures
@pytest.mark.parametrize("path", fixtures(), ids=lambda p: os.path.basename(p))
def test_mps_reader_matches_reference_reader(path):
    """Bit-identical GeneralFormLp, or the same error (class and line)."""
    try:
        ref = O.read_mps(path)
        ref_err = None
    except RuntimeError as e:
        ref, ref_err = None, str(e)
    if ref_err is None:
        assert same_lp(read_mps(path), ref)
    else:
        with pytest.raises((PdlpError, ValueError)) as ei:
            read_mps(path)
        assert str(ei.value).split(": ", 1)[-1] in ref_err or ref_err.split(": ", 1)[-1] in str(ei.value)
        if "line" in ref_err:
            line = ref_err.split("line ")[1].split(":")[0]
            assert f"line {line}:" in str(ei.value)


@needs_fixtures
def test_mps_reader_reproduces_golden_instances():
    suite = ref_suite()
    for name in ("rand01", "transport23", "freevars", "objconst", "infeasible_dual", "tiny2"):
        p = FIX / "suite" / f"{name}.mps"
        if not p.exists():
            p = FIX / f"{name}.mps"
        assert lp_hash(read_mps(p)) == suite[name]["lp_sha256"], name


MPS_TEXT = """NAME          RANGED
ROWS
 N  obj
 L  lim1
 G  lim2
 E  myeqn
 E  eq2
 N  free2
COLUMNS
    x1        obj       1.0        lim1      1.0
    x1        lim2      1.0        free2     4.0
    MARKER    'MARKER'  'INTORG'
    x2        obj       2.0        lim1      1.0
    x2        myeqn     -1.0
    MARKER    'MARKER'  'INTEND'
    x3        obj       -1.0       myeqn     1.0
    x3        eq2       1.0        eq2       2.0
RHS
    rhs       obj       -3.5       lim1      4.0
    rhs       lim2      1.0        myeqn     7.0
    rhs       eq2       2.0
RANGES
    rng       lim1      2.5        myeqn     -2.0
BOUNDS
 UP bnd       x1        4.0
 MI bnd       x2
 BV bnd       x3
ENDATA
"""


def test_parse_mps_semantics_known_answer():
    """docs/mps_format.md: L negated, ranges expanded, E-range < 0, bounds in
    order, extra N rows dropped, objective-row RHS -> -constant, duplicates summed."""
    lp = parse_mps(MPS_TEXT)
    assert lp.objective_constant == 3.5
    assert list(lp.objective) == [1.0, 2.0, -1.0]
    # G rows in declaration order: lim1 (L, ranged: lo 1.5 -> +row, hi 4 -> -row), lim2 (G)
    # myeqn (E, range -2: [5, 7] -> pair)
    G = lp.inequality_matrix.to_dense()
    assert G.tolist() == [[1, 1, 0], [-1, -1, 0], [1, 0, 0], [0, -1, 1], [0, 1, -1]]
    assert list(lp.inequality_rhs) == [1.5, -4.0, 1.0, 5.0, -7.0]
    assert lp.equality_matrix.to_dense().tolist() == [[0, 0, 3.0]]  # eq2: 1 + 2 summed
    assert list(lp.equality_rhs) == [2.0]
    assert list(lp.lower) == [0.0, -np.inf, 0.0] and list(lp.upper) == [4.0, np.inf, 1.0]


def test_parse_mps_errors_carry_line_numbers():
    with pytest.raises(PdlpError, match="line 3: unknown row type 'Q'"):
        parse_mps("NAME X\nROWS\n Q r\nENDATA\n")
    with pytest.raises(PdlpError, match="missing ENDATA"):
        parse_mps("NAME X\nROWS\n N obj\n")
    with pytest.raises(ValueError, match="infeasible bounds on variable 'x'"):
        parse_mps("NAME X\nROWS\n N obj\nCOLUMNS\n x obj 1\nRHS\nBOUNDS\n LO b x 5\n UP b x 2\nENDATA\n")
    with pytest.raises(PdlpError, match="cannot open"):
        read_mps("/nonexistent/file.mps")


def test_fixed_and_free_format_agree():
    def card(f1="", f2="", f3="", f4="", f5="", f6=""):  # fixed columns 2-3, 5-12, 15-22, 25-36, 40-47, 50-61
        return (" " + f1.ljust(2) + " " + f2.ljust(8) + "  " + f3.ljust(8) + "  " + f4.rjust(12) + "   "
                + f5.ljust(8) + "  " + f6.rjust(12)).rstrip()

    fixed = "\n".join(["NAME          T", "ROWS", card("N", "COST"), card("G", "R1"), "COLUMNS",
                       card("", "X 1", "COST", "1.0", "R1", "1.0"), card("", "X2", "COST", "2.0", "R1", "1.0"),
                       "RHS", card("", "RHS", "R1", "1.0"), "ENDATA", ""])
    a = parse_mps(fixed, MPS_FIXED)  # the name "X 1" holds a blank: fixed columns only
    assert a.num_variables == 2 and list(a.objective) == [1.0, 2.0]
    b = parse_mps(fixed.replace("X 1", "X1 "), MPS_FREE)
    assert same_lp(a, b)


def test_gzip_input(tmp_path):
    import gzip

    p = tmp_path / "t.mps.gz"
    p.write_bytes(gzip.compress(MPS_TEXT.encode()))
    assert same_lp(read_mps(p), parse_mps(MPS_TEXT))


def test_write_solution_format(tmp_path):
    """solution_io.hpp:70-95: fixed key order, max_digits10 doubles."""
    from paper_2311_12180_b200.lp import PrimalDualPoint, ReducedCosts, SolveResult, SolveStatus

    info = {"primal_objective": 1.0 / 3.0, "dual_objective": 2.5, "relative_gap": 1e-9,
            "primal_residual_norm": 0.0, "dual_residual_norm": 3e-7}
    r = SolveResult(SolveStatus.OPTIMAL, PrimalDualPoint(np.array([0.1, 2.0]), np.array([-1.5])),
                    ReducedCosts(np.zeros(2), np.zeros(2), np.zeros(2)), info, 42, 1, 0.25)
    p = tmp_path / "s.sol"
    write_solution(r, p, include_vectors=True)
    lines = p.read_text().splitlines()
    assert lines[:9] == ["format_version 1", "status optimal", "primal_objective 0.33333333333333331",
                         "dual_objective 2.5", "relative_gap 1.0000000000000001e-09", "primal_residual 0",
                         "dual_residual 2.9999999999999999e-07", "iterations 42", "solve_seconds 0.25"]
    assert lines[9:] == ["primal_solution 2", "0.10000000000000001", "2", "dual_solution 1", "-1.5"]


def test_cpp_host_header_compiles_and_rejects_bad_input(tmp_path):
    """include/pdlp_b200.hpp (the pdhglp::solve mirror) builds with g++ -std=c++20
    against libpdlp_b200.so; invalid LPs throw std::invalid_argument before any
    device work, and read_mps_file round-trips through the library."""
    src = tmp_path / "t.cpp"
    mps = tmp_path / "t.mps"
    mps.write_text(MPS_TEXT)
    src.write_text(r'''
#include <cstdio>
#include <stdexcept>
#include "pdlp_b200.hpp"
int main(int argc, char** argv) {
  pdlp_b200::GeneralFormLp lp = pdlp_b200::read_mps_file(argv[1]);
  if (lp.num_variables() != 3 || lp.num_inequalities() != 5 || lp.objective_constant != 3.5) return 2;
  lp.lower[1] = 7.0; lp.upper[1] = 6.0;  // crossing bounds
  try { pdlp_b200::solve(lp); return 3; } catch (const std::invalid_argument& e) {
    std::printf("invalid_argument: %s\n", e.what()); }
  pdlp_b200::SolverParams p; p.beta_sufficient = 0.9;
  try { p.validate(); return 4; } catch (const std::invalid_argument&) {}
  try { pdlp_b200::read_mps_file("/nonexistent.mps"); return 5; } catch (const std::runtime_error&) {}
  std::printf("ok\n");
  return 0;
}
''')
    lib = library_path()
    exe = tmp_path / "t"
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", str(ROOT / "include"), str(src), "-o", str(exe),
                    str(lib), f"-Wl,-rpath,{lib.parent}"], check=True)
    out = subprocess.run([str(exe), str(mps)], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "empty bound interval on variable 1" in out.stdout and out.stdout.endswith("ok\n")
