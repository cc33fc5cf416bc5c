"""Python binding of the C-ABI (include/pdlp_b200.h) — the B200 solver.

`solve(lp, params)` is the drop-in for pdhglp::solve (solver.hpp:935-940);
`Solver` keeps the instance resident in HBM across calls and exposes the
kernel-level entry points (spmv, scaling, stepwise iteration) the parity tests
use. Everything here calls libpdlp_b200.so; there is no CPU fallback — a
missing library or GPU raises.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

from . import abi
from .lp import GeneralFormLp, SolveResult, SolverParams, result_from_buffers

_LIB_PATH = Path(__file__).resolve().parent / "lib" / "libpdlp_b200.so"
_lib = None


class PdlpError(RuntimeError):
    pass


def library_path() -> Path:
    return _LIB_PATH


def load_library(build_if_missing: bool = True) -> C.CDLL:
    """Loads the in-tree libpdlp_b200.so (building it with nvcc if absent)."""
    global _lib
    if _lib is not None:
        return _lib
    if not _LIB_PATH.exists() and build_if_missing:
        from . import _build

        _build.build()
    if not _LIB_PATH.exists():
        raise PdlpError(f"CUDA library missing: {_LIB_PATH} (run __graft_entry__.build())")
    lib = C.CDLL(str(_LIB_PATH))
    H = C.c_void_p
    dp, i64p, i32p = C.POINTER(C.c_double), C.POINTER(C.c_int64), C.POINTER(C.c_int32)
    sig = {
        "pdlp_abi_version": (C.c_int, []),
        "pdlp_default_params": (None, [C.POINTER(abi.PdlpParams)]),
        "pdlp_create": (C.c_int, [C.POINTER(abi.PdlpLp), C.POINTER(abi.PdlpParams), C.POINTER(H)]),
        "pdlp_destroy": (None, [H]),
        "pdlp_solve": (C.c_int, [H, C.POINTER(abi.PdlpResultInfo)]),
        "pdlp_get_solution": (C.c_int, [H, dp, dp, dp, dp, dp]),
        "pdlp_get_step_log": (C.c_int, [H, C.c_void_p, C.c_int64]),
        "pdlp_get_restart_log": (C.c_int, [H, C.c_void_p, C.c_int64]),
        "pdlp_get_scaling": (C.c_int, [H, dp, dp]),
        "pdlp_spmv": (C.c_int, [H, C.c_int32, dp, dp]),
        "pdlp_iterate_begin": (C.c_int, [H, i32p]),
        "pdlp_iterate_run": (C.c_int, [H, C.c_int64, i32p]),
        "pdlp_get_iterate": (C.c_int, [H, dp, dp, dp, dp, i64p, dp]),
        "pdlp_time_kernel": (C.c_int, [H, C.c_int32, C.c_int32, dp, dp]),
        "pdlp_get_sizes": (C.c_int, [H, i64p]),
        "pdlp_last_error": (C.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    if lib.pdlp_abi_version() != 1:
        raise PdlpError("ABI version mismatch")
    _lib = lib
    return lib


def _check(rc: int) -> None:
    if rc == abi.PDLP_OK:
        return
    msg = _lib.pdlp_last_error().decode(errors="replace")
    if rc == abi.PDLP_EINVAL:
        raise ValueError(msg)
    raise PdlpError(f"pdlp error {rc}: {msg}")


def default_params() -> abi.PdlpParams:
    lib = load_library()
    p = abi.PdlpParams()
    lib.pdlp_default_params(C.byref(p))
    return p


class Solver:
    """One device-resident instance (pdlp_create ... pdlp_destroy)."""

    def __init__(self, lp: GeneralFormLp, params: SolverParams | None = None):
        self._lib = load_library()
        self.params = params or SolverParams()
        self._lp = lp  # keeps the host arrays alive during create
        self._h = C.c_void_p()
        lpa = lp.to_abi()
        pa = self.params.to_abi()
        _check(self._lib.pdlp_create(C.byref(lpa), C.byref(pa), C.byref(self._h)))
        sizes = np.zeros(4, np.int64)
        _check(self._lib.pdlp_get_sizes(self._h, abi.i64ptr(sizes)))
        self.n, self.m, self.m1, self.nnz = (int(v) for v in sizes)
        self.last_info: abi.PdlpResultInfo | None = None

    def close(self) -> None:
        if self._h:
            self._lib.pdlp_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # ---- whole solve ----
    def solve(self) -> SolveResult:
        info = abi.PdlpResultInfo()
        _check(self._lib.pdlp_solve(self._h, C.byref(info)))
        self.last_info = info
        return self.result()

    def result(self) -> SolveResult:
        info = self.last_info
        n, m = self.n, self.m
        x, y = np.zeros(n), np.zeros(m)
        lam, pos, neg = np.zeros(n), np.zeros(n), np.zeros(n)
        _check(self._lib.pdlp_get_solution(self._h, *(abi.dptr(a) for a in (x, y, lam, pos, neg))))
        slog = np.zeros(info.step_log_size, abi.STEP_LOG_DTYPE)
        rlog = np.zeros(info.restart_log_size, abi.RESTART_DTYPE)
        if slog.size:
            _check(self._lib.pdlp_get_step_log(self._h, slog.ctypes.data, slog.size))
        if rlog.size:
            _check(self._lib.pdlp_get_restart_log(self._h, rlog.ctypes.data, rlog.size))
        return result_from_buffers(info, x, y, lam, pos, neg, slog, rlog)

    # ---- kernel-level entry points ----
    def spmv(self, op: int, v: np.ndarray) -> np.ndarray:
        v = np.ascontiguousarray(v, dtype=np.float64)
        out = np.zeros(self.n if op in (abi.OP_KT_SCALED, abi.OP_KT_ORIGINAL) else self.m)
        _check(self._lib.pdlp_spmv(self._h, op, abi.dptr(v), abi.dptr(out)))
        return out

    def scaling(self) -> tuple[np.ndarray, np.ndarray]:
        d1, d2 = np.zeros(self.m), np.zeros(self.n)
        _check(self._lib.pdlp_get_scaling(self._h, abi.dptr(d1), abi.dptr(d2)))
        return d1, d2

    def iterate_begin(self) -> int:
        st = C.c_int32()
        _check(self._lib.pdlp_iterate_begin(self._h, C.byref(st)))
        return st.value

    def iterate_run(self, n: int) -> int:
        st = C.c_int32()
        _check(self._lib.pdlp_iterate_run(self._h, int(n), C.byref(st)))
        return st.value

    def iterate(self) -> dict:
        x, y, kx, kty = np.zeros(self.n), np.zeros(self.m), np.zeros(self.m), np.zeros(self.n)
        cnt, sc = np.zeros(4, np.int64), np.zeros(4)
        _check(
            self._lib.pdlp_get_iterate(
                self._h, *(abi.dptr(a) for a in (x, y, kx, kty)), abi.i64ptr(cnt), abi.dptr(sc)
            )
        )
        return {
            "x": x, "y": y, "kx": kx, "kty": kty,
            "total": int(cnt[0]), "inner": int(cnt[1]), "outer": int(cnt[2]), "trials": int(cnt[3]),
            "eta": sc[0], "eta_hat": sc[1], "omega": sc[2], "weight_sum": sc[3],
        }

    def time_kernel(self, which: int, reps: int = 50) -> tuple[float, float]:
        ms, by = C.c_double(), C.c_double()
        _check(self._lib.pdlp_time_kernel(self._h, which, reps, C.byref(ms), C.byref(by)))
        return ms.value, by.value


def solve(lp: GeneralFormLp, params: SolverParams | None = None) -> SolveResult:
    """pdhglp::solve (solver.hpp:935-940) on the GPU."""
    lp.validate()
    (params or SolverParams()).validate()
    with Solver(lp, params) as s:
        return s.solve()


__all__ = ["Solver", "solve", "load_library", "default_params", "PdlpError", "library_path"]
