"""CPU tests (no GPU) of the product's host side: the C-ABI library loads and
exports every entry point include/pdlp_b200.h declares, defaults mirror
SolverParams (solver.hpp:59-77), invalid input is rejected with the
reference's error class before any device work, and the seeded generators
produce the BASELINE.json shapes."""
from __future__ import annotations

import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2311_12180_b200 import CsrMatrix, GeneralFormLp, SolverParams, abi, api, generators
from paper_2311_12180_b200.api import load_library

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "pdlp_b200.h"


def declared_symbols() -> list[str]:
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|void|const char\*|const pdlp_lp\*)\s+(pdlp_\w+)\s*\(", text, flags=re.M)))


def test_library_exports_every_declared_symbol():
    syms = declared_symbols()
    assert len(syms) >= 15
    lib = C.CDLL(str(api.library_path()))
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_library_is_sm100a_and_exports_only_c_abi():
    """The product .so carries sm_100a SASS (cross-compiled here)."""
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(api.library_path())],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    nm = subprocess.run(["nm", "-D", "--defined-only", str(api.library_path())], capture_output=True,
                        text=True).stdout
    exported = sorted({ln.split()[-1] for ln in nm.splitlines() if " T " in ln and ln.split()[-1].startswith("pdlp_")})
    assert exported == declared_symbols()


def test_abi_struct_layout_matches_header():
    """ctypes mirror sizes (abi.py) equal the C struct sizes: compile a probe."""
    import subprocess
    import tempfile

    src = r'''
#include <stdio.h>
#include "pdlp_b200.h"
int main(void) { printf("%zu %zu %zu %zu %zu %zu\n", sizeof(pdlp_csr), sizeof(pdlp_lp), sizeof(pdlp_params),
  sizeof(pdlp_result_info), sizeof(pdlp_step_log_entry), sizeof(pdlp_restart_event)); return 0; }
'''
    with tempfile.TemporaryDirectory() as d:
        (Path(d) / "p.c").write_text(src)
        subprocess.run(["gcc", "-I", str(ROOT / "include"), "-o", f"{d}/p", f"{d}/p.c"], check=True)
        sizes = [int(v) for v in subprocess.run([f"{d}/p"], capture_output=True, text=True).stdout.split()]
    assert sizes == [C.sizeof(abi.PdlpCsr), C.sizeof(abi.PdlpLp), C.sizeof(abi.PdlpParams),
                     C.sizeof(abi.PdlpResultInfo), abi.STEP_LOG_DTYPE.itemsize, abi.RESTART_DTYPE.itemsize]


def test_default_params_mirror_reference_defaults():
    lib = load_library()
    assert lib.pdlp_abi_version() == 1
    p = abi.PdlpParams()
    lib.pdlp_default_params(C.byref(p))
    py = SolverParams()
    for name, _ in abi.PdlpParams._fields_:
        if name == "reserved":
            continue
        assert getattr(p, name) == int(getattr(py, name)) if isinstance(getattr(py, name), (bool, int)) \
            else getattr(p, name) == getattr(py, name), name
    # solver.hpp:59-77
    assert (p.eps_optimal, p.eps_infeasible, p.evaluation_frequency, p.ruiz_iterations) == (1e-4, 1e-8, 64, 10)
    assert (p.beta_sufficient, p.beta_necessary, p.beta_artificial, p.theta_smoothing) == (0.2, 0.8, 0.36, 0.5)
    assert (p.step_reduction_exponent, p.step_growth_exponent, p.omega_min, p.omega_max) == (0.3, 0.6, 1e-8, 1e8)


def _tiny_lp(**kw) -> GeneralFormLp:
    G = CsrMatrix.from_triplets(1, 2, [0, 0], [0, 1], [1.0, 1.0])
    d = dict(inequality_matrix=G, equality_matrix=CsrMatrix.zero(0, 2), objective=[1.0, 1.0],
             inequality_rhs=[1.0], equality_rhs=np.zeros(0), lower=[0.0, 0.0], upper=[10.0, 10.0])
    d.update(kw)
    return GeneralFormLp(**d)


@pytest.mark.parametrize("bad, msg", [
    (dict(lower=[0.0, np.nan]), "NaN bound on variable 1"),
    (dict(lower=[0.0, 5.0], upper=[10.0, 4.0]), "empty bound interval on variable 1"),
    (dict(lower=[np.inf, 0.0], upper=[np.inf, 1.0]), "empty bound interval on variable 0"),
    (dict(objective=[1.0, np.nan]), "NaN objective"),
])
def test_invalid_lp_is_einval_before_device_work(bad, msg):
    """lp_model.hpp:45-72 throws std::invalid_argument; the C-ABI returns
    PDLP_EINVAL (raised as ValueError) without touching the GPU."""
    lp = _tiny_lp(**bad)
    with pytest.raises(ValueError, match=msg):
        lp.validate()
    lib = load_library()
    h = C.c_void_p()
    lpa, pa = lp.to_abi(), SolverParams().to_abi()
    rc = lib.pdlp_create(C.byref(lpa), C.byref(pa), C.byref(h))
    assert rc == abi.PDLP_EINVAL
    assert msg in lib.pdlp_last_error().decode()
    assert not h.value


@pytest.mark.parametrize("field, value", [("eps_optimal", 0.0), ("beta_sufficient", 0.9),
                                          ("theta_smoothing", 1.5), ("evaluation_frequency", 0)])
def test_invalid_params_is_einval(field, value):
    """SolverParams::validate (solver.hpp:79-93)."""
    p = SolverParams(**{field: value})
    with pytest.raises(ValueError):
        p.validate()
    lib = load_library()
    h = C.c_void_p()
    lpa, pa = _tiny_lp().to_abi(), p.to_abi()
    assert lib.pdlp_create(C.byref(lpa), C.byref(pa), C.byref(h)) == abi.PDLP_EINVAL


def test_null_handle_calls_fail_cleanly():
    lib = load_library()
    info = abi.PdlpResultInfo()
    assert lib.pdlp_solve(None, C.byref(info)) == abi.PDLP_EINVAL
    assert lib.pdlp_last_error() == b"null handle"
    lib.pdlp_destroy(None)


def test_no_cpu_fallback_in_product_path():
    """The product package never imports the oracle (test infrastructure)."""
    pkg = ROOT / "paper_2311_12180_b200"
    for f in pkg.rglob("*.py"):
        assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\w+)", f.read_text(), flags=re.M), f


def test_generator_shapes():
    c1 = generators.config("C1")
    assert (c1.num_constraints, c1.num_variables, c1.nnz, c1.num_inequalities) == (10000, 20000, 100000, 5000)
    t = generators.transport_lp(20, 30, seed=1)
    assert (t.num_constraints, t.num_variables, t.nnz) == (50, 600, 1200)
    assert t.equality_rhs[:20].sum() == t.equality_rhs[20:].sum()
    # every column of the transport LP has exactly one supply and one demand row
    col_counts = np.bincount(t.equality_matrix.col_indices, minlength=600)
    assert (col_counts == 2).all()
    # C1 rows are sorted/unique per row (CsrMatrix invariants, sparse_matrix.hpp:29-34)
    K = c1.equality_matrix
    for r in range(0, K.num_rows, 997):
        cols = K.col_indices[K.row_offsets[r]:K.row_offsets[r + 1]]
        assert (np.diff(cols) > 0).all()


def test_generator_is_deterministic():
    a, b = generators.random_lp(50, 40, 120, 3, seed=7), generators.random_lp(50, 40, 120, 3, seed=7)
    assert np.array_equal(a.equality_matrix.values, b.equality_matrix.values)
    assert np.array_equal(a.inequality_rhs, b.inequality_rhs)
