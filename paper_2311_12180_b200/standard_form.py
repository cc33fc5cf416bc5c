"""Standard-form theory harness on the B200 (standard_form.hpp:36-211; SURVEY.md
section 8f, rank 4), with the reference's names:

* StandardFormLp              min c'x s.t. Ax = b, x >= 0 (standard_form.hpp:18-33)
* kkt_error_standard          ||(Ax - b; [-x]+; [A'y - c]+; [c'x - b'y]+)|| (:37-58)
* spectral_norm               power iteration on A'A (:63-89)
* p_s_norm_squared            ||x||^2 + ||y||^2 + 2 s y'Ax (:92-98)
* StandardPdhgOptions / StandardEpoch / StandardPdhgTrace (:100-128)
* restarted_pdhg_standard     fixed-step PDHG, uniform averages, restart to the
                              average once KKT(avg) <= beta KKT(epoch start) (:131-211)

Everything runs in the GPU library (csrc/standard_form.cu). `parity=True`
keeps the reference's summation order (bitwise results); the default fast mode
uses the tiled SpMV engine and tree sums.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import abi
from .lp import CsrMatrix, PrimalDualPoint


@dataclass
class StandardFormLp:
    constraint_matrix: CsrMatrix  # A, m x n
    rhs: np.ndarray               # b
    objective: np.ndarray         # c

    @property
    def num_variables(self) -> int:
        return self.constraint_matrix.num_cols

    @property
    def num_constraints(self) -> int:
        return self.constraint_matrix.num_rows

    def validate(self) -> None:
        if len(self.rhs) != self.num_constraints or len(self.objective) != self.num_variables:
            raise ValueError("standard-form lp: dimension mismatch")


@dataclass
class StandardPdhgOptions:
    step_size: float = 0.0         # s; both primal and dual step
    restart_decay: float = 0.5     # beta in (0, 1)
    convergence_tol: float = 1e-9  # stop once the epoch-start KKT error drops below
    iteration_limit: int = 1_000_000
    record_iterates: bool = False  # keep every inner iterate per epoch
    # B200 extensions
    parity: bool = False
    device: int = 0

    def validate(self) -> None:
        if not (self.step_size > 0.0):
            raise ValueError("step_size must be positive")
        if not (0.0 < self.restart_decay < 1.0):
            raise ValueError("restart_decay must lie in (0, 1)")


@dataclass
class StandardEpoch:
    start: PrimalDualPoint | None
    start_kkt: float = 0.0
    length: int = 0
    iterates: list[PrimalDualPoint] = field(default_factory=list)


@dataclass
class StandardPdhgTrace:
    epochs: list[StandardEpoch] = field(default_factory=list)
    total_iterations: int = 0
    converged: bool = False
    numerical_failure: bool = False


class _Csr:
    """Keeps the int64 / f64 arrays alive behind a pdlp_csr."""

    def __init__(self, a: CsrMatrix):
        self.off = np.ascontiguousarray(a.row_offsets, dtype=np.int64)
        self.col = np.ascontiguousarray(a.col_indices, dtype=np.int64)
        self.val = np.ascontiguousarray(a.values, dtype=np.float64)
        self.c = abi.PdlpCsr(num_rows=a.num_rows, num_cols=a.num_cols, nnz=len(self.val),
                             row_offsets=abi.i64ptr(self.off), col_indices=abi.i64ptr(self.col),
                             values=abi.dptr(self.val))


def _lib():
    from .api import load_library

    lib = load_library()
    if not getattr(lib, "_sf_bound", False):
        dp, i64p = C.POINTER(C.c_double), C.POINTER(C.c_int64)
        CP = C.POINTER(abi.PdlpCsr)
        lib.pdlp_standard_default_options.argtypes = [C.POINTER(abi.PdlpStandardOptions)]
        lib.pdlp_standard_default_options.restype = None
        lib.pdlp_standard_pdhg.argtypes = [CP, dp, dp, C.POINTER(abi.PdlpStandardOptions), dp, dp, dp, i64p,
                                           C.c_int64, i64p, dp, dp, dp, dp, C.c_int64]
        lib.pdlp_kkt_error_standard.argtypes = [CP, dp, dp, dp, dp, C.c_int32, C.c_int32, dp]
        lib.pdlp_spectral_norm.argtypes = [CP, C.c_double, C.c_int32, C.c_int32, C.c_int32, dp]
        lib.pdlp_p_s_norm_squared.argtypes = [CP, dp, dp, C.c_double, dp, dp, C.c_int32, C.c_int32, dp]
        lib._sf_bound = True
    return lib


def _f64(v) -> np.ndarray:
    return np.ascontiguousarray(v, dtype=np.float64)


def _check(rc: int) -> None:
    from .api import _check as check

    check(rc)


def kkt_error_standard(lp: StandardFormLp, x, y, *, parity: bool = False, device: int = 0) -> float:
    a = _Csr(lp.constraint_matrix)
    b, c, xv, yv = _f64(lp.rhs), _f64(lp.objective), _f64(x), _f64(y)
    out = C.c_double(0.0)
    _check(_lib().pdlp_kkt_error_standard(C.byref(a.c), abi.dptr(b), abi.dptr(c), abi.dptr(xv), abi.dptr(yv),
                                          int(parity), device, C.byref(out)))
    return out.value


def spectral_norm(a: CsrMatrix, tol: float = 1e-10, max_iterations: int = 10000, *, parity: bool = False,
                  device: int = 0) -> float:
    m = _Csr(a)
    out = C.c_double(0.0)
    _check(_lib().pdlp_spectral_norm(C.byref(m.c), tol, max_iterations, int(parity), device, C.byref(out)))
    return out.value


def p_s_norm_squared(lp: StandardFormLp, step_size: float, x, y, *, parity: bool = False, device: int = 0) -> float:
    a = _Csr(lp.constraint_matrix)
    b, c, xv, yv = _f64(lp.rhs), _f64(lp.objective), _f64(x), _f64(y)
    out = C.c_double(0.0)
    _check(_lib().pdlp_p_s_norm_squared(C.byref(a.c), abi.dptr(b), abi.dptr(c), step_size, abi.dptr(xv),
                                        abi.dptr(yv), int(parity), device, C.byref(out)))
    return out.value


def restarted_pdhg_standard(lp: StandardFormLp, options: StandardPdhgOptions,
                            start: PrimalDualPoint | None = None, *, max_epochs: int = 1 << 16,
                            max_recorded: int = 1 << 16) -> StandardPdhgTrace:
    """The GPU run of restarted_pdhg_standard. Epoch start points other than
    the first and the last are not kept (the device does not store them);
    with record_iterates, the first `max_recorded` iterates are returned,
    split into their epochs."""
    lp.validate()
    options.validate()
    n, m = lp.num_variables, lp.num_constraints
    a = _Csr(lp.constraint_matrix)
    b, c = _f64(lp.rhs), _f64(lp.objective)
    o = abi.PdlpStandardOptions()
    _lib().pdlp_standard_default_options(C.byref(o))
    o.step_size, o.restart_decay, o.convergence_tol = options.step_size, options.restart_decay, options.convergence_tol
    o.iteration_limit, o.parity, o.device = options.iteration_limit, int(options.parity), options.device
    x0 = y0 = None
    if start is not None and len(start.primal):
        x0, y0 = _f64(start.primal), _f64(start.dual)
    kkt = np.zeros(max_epochs)
    lens = np.zeros(max_epochs, np.int64)
    cnt = np.zeros(4, np.int64)
    xl, yl = np.zeros(n), np.zeros(m)
    cap_it = max_recorded if options.record_iterates else 0
    ix, iy = np.zeros(max(cap_it, 1) * n), np.zeros(max(cap_it, 1) * m)
    _check(_lib().pdlp_standard_pdhg(
        C.byref(a.c), abi.dptr(b), abi.dptr(c), C.byref(o), abi.dptr(x0) if x0 is not None else None,
        abi.dptr(y0) if y0 is not None else None, abi.dptr(kkt), abi.i64ptr(lens), max_epochs, abi.i64ptr(cnt),
        abi.dptr(xl), abi.dptr(yl), abi.dptr(ix) if cap_it else None, abi.dptr(iy) if cap_it else None, cap_it))
    ne = int(cnt[0])
    tr = StandardPdhgTrace(total_iterations=int(cnt[1]), converged=bool(cnt[2]), numerical_failure=bool(cnt[3]))
    first = PrimalDualPoint(x0.copy(), y0.copy()) if x0 is not None else PrimalDualPoint(np.zeros(n), np.zeros(m))
    k = 0
    for e in range(min(ne, max_epochs)):
        ep = StandardEpoch(start=first if e == 0 else None, start_kkt=float(kkt[e]), length=int(lens[e]))
        if cap_it:
            for _ in range(ep.length):
                if k >= min(cap_it, tr.total_iterations):
                    break
                ep.iterates.append(PrimalDualPoint(ix[k * n:(k + 1) * n].copy(), iy[k * m:(k + 1) * m].copy()))
                k += 1
        tr.epochs.append(ep)
    if tr.epochs:
        tr.epochs[-1].start = PrimalDualPoint(xl, yl)
    return tr
