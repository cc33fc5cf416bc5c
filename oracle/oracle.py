"""TEST INFRASTRUCTURE ONLY — ctypes bindings of the CPU checkers.

  kind="oracle": oracle/_build/liboracle.so   (plain-C restatement, pdlp_oracle.c)
  kind="ref":    oracle/_ref/libpdhglp_ref.so (the reference headers compiled in place)

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this. The
product (paper_2311_12180_b200, libpdlp_b200.so) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

from paper_2311_12180_b200 import abi
from paper_2311_12180_b200.lp import CsrMatrix, GeneralFormLp, SolverParams, result_from_buffers

HERE = Path(__file__).resolve().parent
PATHS = {
    "oracle": HERE / "_build" / "liboracle.so",
    "ref": HERE / "_ref" / "libpdhglp_ref.so",
}
PREFIX = {"oracle": "oracle_", "ref": "ref_"}
_libs: dict[str, C.CDLL] = {}


def available(kind: str) -> bool:
    return PATHS[kind].exists()


def build(kind: str = "oracle") -> None:
    target = {"oracle": "oracle", "ref": "ref"}[kind]
    subprocess.run(["make", "-s", "-C", str(HERE), target], check=True)


def load(kind: str = "oracle") -> C.CDLL:
    if kind in _libs:
        return _libs[kind]
    if not PATHS[kind].exists():
        if kind == "oracle":
            build("oracle")
        else:
            raise FileNotFoundError(f"{PATHS[kind]} not built (needs /root/reference)")
    lib = C.CDLL(str(PATHS[kind]))
    p = PREFIX[kind]
    dp, i64p, i32p = C.POINTER(C.c_double), C.POINTER(C.c_int64), C.POINTER(C.c_int32)
    LPP, PP = C.POINTER(abi.PdlpLp), C.POINTER(abi.PdlpParams)
    sigs = {
        "solve": (C.c_int, [LPP, PP, C.POINTER(abi.PdlpResultInfo), dp, dp, dp, dp, dp,
                            C.c_void_p, C.c_int64, C.c_void_p, C.c_int64]),
        "begin": (C.c_void_p, [LPP, PP, i32p]),
        "run": (C.c_int, [C.c_void_p, C.c_int64, i32p]),
        "get_iterate": (C.c_int, [C.c_void_p, dp, dp, dp, dp, i64p, dp]),
        "result": (C.c_int, [C.c_void_p, C.POINTER(abi.PdlpResultInfo), dp, dp, dp, dp, dp,
                             C.c_void_p, C.c_int64, C.c_void_p, C.c_int64]),
        "end": (None, [C.c_void_p]),
        "scaling": (C.c_int, [LPP, PP, dp, dp]),
        "spmv": (C.c_int, [C.POINTER(abi.PdlpCsr), dp, dp]),
        "spmv_transpose": (C.c_int, [C.POINTER(abi.PdlpCsr), dp, dp]),
        "transpose": (C.c_int, [C.POINTER(abi.PdlpCsr), i64p, i64p, dp]),
        "from_triplets": (C.c_int, [C.c_int64, C.c_int64, C.c_int64, i64p, i64p, dp, i64p, i64p,
                                    dp, i64p]),
        "last_error": (C.c_char_p, []),
        "check_termination": (C.c_int, [LPP, dp, dp, C.c_double, dp]),
        "pdhg_raw_step": (C.c_int, [LPP, dp, dp, C.c_double, C.c_double, dp, dp]),
    }
    for name, (res, args) in sigs.items():
        f = getattr(lib, p + name)
        f.restype = res
        f.argtypes = args
    if kind == "ref":
        lib.ref_mps_load.restype = C.c_void_p
        lib.ref_mps_load.argtypes = [C.c_char_p]
        lib.ref_mps_sizes.argtypes = [C.c_void_p, i64p]
        lib.ref_mps_fill.argtypes = [C.c_void_p, i64p, i64p, dp, i64p, i64p, dp, dp, dp, dp, dp, dp, dp]
        lib.ref_mps_free.argtypes = [C.c_void_p]
    _libs[kind] = lib
    return lib


def set_sum_order(order: int) -> None:
    """Summation-order probe of the C restatement (0: the reference's
    sequential step-size sums; 1: pairwise trees). Process-wide."""
    lib = load("oracle")
    lib.oracle_set_sum_order.argtypes = [C.c_int]
    lib.oracle_set_sum_order.restype = None
    lib.oracle_set_sum_order(int(order))


def _f(lib, kind, name):
    return getattr(lib, PREFIX[kind] + name)


def _err(lib, kind, rc):
    if rc != 0:
        msg = _f(lib, kind, "last_error")().decode(errors="replace")
        if rc == abi.PDLP_EINVAL:
            raise ValueError(msg)
        raise RuntimeError(f"{kind} error {rc}: {msg}")


def solve(lp: GeneralFormLp, params: SolverParams | None = None, kind: str = "oracle",
          log_capacity: int = 2_000_000):
    params = params or SolverParams()
    lib = load(kind)
    lpa, pa = lp.to_abi(), params.to_abi()
    info = abi.PdlpResultInfo()
    n, m = lp.num_variables, lp.num_constraints
    x, y, lam, pos, neg = np.zeros(n), np.zeros(m), np.zeros(n), np.zeros(n), np.zeros(n)
    cap = log_capacity if params.record_step_log else 0
    slog = np.zeros(cap, abi.STEP_LOG_DTYPE)
    rlog = np.zeros(100_000, abi.RESTART_DTYPE)
    rc = _f(lib, kind, "solve")(C.byref(lpa), C.byref(pa), C.byref(info),
                                *(abi.dptr(a) for a in (x, y, lam, pos, neg)),
                                slog.ctypes.data if cap else None, cap, rlog.ctypes.data, rlog.size)
    _err(lib, kind, rc)
    return result_from_buffers(info, x, y, lam, pos, neg, slog[: min(cap, info.step_log_size)],
                               rlog[: info.restart_log_size])


class Session:
    """Stepwise loop: oracle_/ref_ begin, run, get_iterate, result, end."""

    def __init__(self, lp: GeneralFormLp, params: SolverParams | None = None, kind: str = "oracle"):
        self.kind, self.lib = kind, load(kind)
        self.params = params or SolverParams()
        self._lp = lp
        self.n, self.m = lp.num_variables, lp.num_constraints
        st = C.c_int32()
        lpa, pa = lp.to_abi(), self.params.to_abi()
        self.h = _f(self.lib, kind, "begin")(C.byref(lpa), C.byref(pa), C.byref(st))
        if not self.h:
            raise ValueError(_f(self.lib, kind, "last_error")().decode())
        self.status = st.value

    def run(self, k: int) -> int:
        st = C.c_int32()
        _err(self.lib, self.kind, _f(self.lib, self.kind, "run")(self.h, int(k), C.byref(st)))
        self.status = st.value
        return st.value

    def fork(self) -> "Session":
        """An independent copy of the iterate state sharing the read-only setup
        (reference harness only)."""
        if self.kind != "ref":
            raise ValueError("fork: reference sessions only")
        fn = self.lib.ref_fork
        fn.restype, fn.argtypes = C.c_void_p, [C.c_void_p]
        s = Session.__new__(Session)
        s.kind, s.lib, s.params, s._lp, s.n, s.m, s.status = self.kind, self.lib, self.params, self._lp, \
            self.n, self.m, self.status
        s.h = fn(self.h)
        if not s.h:
            raise RuntimeError(_f(self.lib, self.kind, "last_error")().decode())
        return s

    def iterate(self) -> dict:
        x, y, kx, kty = np.zeros(self.n), np.zeros(self.m), np.zeros(self.m), np.zeros(self.n)
        cnt, sc = np.zeros(4, np.int64), np.zeros(4)
        _f(self.lib, self.kind, "get_iterate")(self.h, *(abi.dptr(a) for a in (x, y, kx, kty)),
                                               abi.i64ptr(cnt), abi.dptr(sc))
        return {"x": x, "y": y, "kx": kx, "kty": kty, "total": int(cnt[0]), "inner": int(cnt[1]),
                "outer": int(cnt[2]), "trials": int(cnt[3]), "eta": sc[0], "eta_hat": sc[1],
                "omega": sc[2], "weight_sum": sc[3]}

    def result(self):
        info = abi.PdlpResultInfo()
        n, m = self.n, self.m
        x, y, lam, pos, neg = np.zeros(n), np.zeros(m), np.zeros(n), np.zeros(n), np.zeros(n)
        _err(self.lib, self.kind, _f(self.lib, self.kind, "result")(
            self.h, C.byref(info), *(abi.dptr(a) for a in (x, y, lam, pos, neg)), None, 0, None, 0))
        return result_from_buffers(info, x, y, lam, pos, neg, np.zeros(0, abi.STEP_LOG_DTYPE),
                                   np.zeros(0, abi.RESTART_DTYPE))

    def close(self):
        if self.h:
            _f(self.lib, self.kind, "end")(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def scaling(lp: GeneralFormLp, params: SolverParams | None = None, kind: str = "oracle"):
    params = params or SolverParams()
    lib = load(kind)
    d1, d2 = np.zeros(lp.num_constraints), np.zeros(lp.num_variables)
    lpa, pa = lp.to_abi(), params.to_abi()
    _err(lib, kind, _f(lib, kind, "scaling")(C.byref(lpa), C.byref(pa), abi.dptr(d1), abi.dptr(d2)))
    return d1, d2


def spmv(a: CsrMatrix, x, kind: str = "oracle") -> np.ndarray:
    lib = load(kind)
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.zeros(a.num_rows)
    ca = a.to_abi()
    _err(lib, kind, _f(lib, kind, "spmv")(C.byref(ca), abi.dptr(x), abi.dptr(out)))
    return out


def spmv_transpose(a: CsrMatrix, y, kind: str = "oracle") -> np.ndarray:
    lib = load(kind)
    y = np.ascontiguousarray(y, dtype=np.float64)
    out = np.zeros(a.num_cols)
    ca = a.to_abi()
    _err(lib, kind, _f(lib, kind, "spmv_transpose")(C.byref(ca), abi.dptr(y), abi.dptr(out)))
    return out


def transpose(a: CsrMatrix, kind: str = "oracle") -> CsrMatrix:
    lib = load(kind)
    off, col, val = np.zeros(a.num_cols + 1, np.int64), np.zeros(a.nnz, np.int64), np.zeros(a.nnz)
    ca = a.to_abi()
    _err(lib, kind, _f(lib, kind, "transpose")(C.byref(ca), abi.i64ptr(off), abi.i64ptr(col), abi.dptr(val)))
    return CsrMatrix(a.num_cols, a.num_rows, off, col, val)


def from_triplets(rows: int, cols: int, r, c, v, kind: str = "oracle") -> CsrMatrix:
    lib = load(kind)
    r = np.ascontiguousarray(r, dtype=np.int64)
    c = np.ascontiguousarray(c, dtype=np.int64)
    v = np.ascontiguousarray(v, dtype=np.float64)
    off, col, val = np.zeros(rows + 1, np.int64), np.zeros(r.size, np.int64), np.zeros(r.size)
    nnz = C.c_int64()
    _err(lib, kind, _f(lib, kind, "from_triplets")(rows, cols, r.size, abi.i64ptr(r), abi.i64ptr(c),
                                                    abi.dptr(v), abi.i64ptr(off), abi.i64ptr(col),
                                                    abi.dptr(val), C.byref(nnz)))
    k = nnz.value
    return CsrMatrix(rows, cols, off, col[:k].copy(), val[:k].copy())


def check_termination(lp: GeneralFormLp, x, y, eps: float, kind: str = "oracle") -> dict:
    """The reference's own criteria recomputed at a returned point (criterion 2 style)."""
    lib = load(kind)
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    out = np.zeros(5)
    lpa = lp.to_abi()
    _err(lib, kind, _f(lib, kind, "check_termination")(C.byref(lpa), abi.dptr(x), abi.dptr(y), eps, abi.dptr(out)))
    return {"terminated": bool(out[0]), "primal_residual_norm": out[1], "dual_residual_norm": out[2],
            "primal_objective_raw": out[3], "dual_objective_raw": out[4]}


def pdhg_raw_step(lp: GeneralFormLp, x, y, tau: float, sigma: float, kind: str = "oracle"):
    """pdhg_raw_step (solver.hpp:335-358) on to_saddle(lp): returns (x', y')."""
    lib = load(kind)
    lpa = lp.to_abi()
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    xo, yo = np.empty(lp.num_variables), np.empty(lp.num_constraints)
    dp = C.POINTER(C.c_double)
    _err(lib, kind, _f(lib, kind, "pdhg_raw_step")(C.byref(lpa), x.ctypes.data_as(dp), y.ctypes.data_as(dp),
                                                 float(tau), float(sigma), xo.ctypes.data_as(dp),
                                                 yo.ctypes.data_as(dp)))
    return xo, yo


def read_mps(path: str | os.PathLike) -> GeneralFormLp:
    """The reference's own MPS reader (mps_io.hpp:582) — fixture generation only."""
    lib = load("ref")
    h = lib.ref_mps_load(str(path).encode())
    if not h:
        raise RuntimeError(lib.ref_last_error().decode())
    sz = np.zeros(5, np.int64)
    lib.ref_mps_sizes(h, abi.i64ptr(sz))
    n, m1, m2, ng, na = (int(v) for v in sz)
    g_off, g_col, g_val = np.zeros(m1 + 1, np.int64), np.zeros(ng, np.int64), np.zeros(ng)
    a_off, a_col, a_val = np.zeros(m2 + 1, np.int64), np.zeros(na, np.int64), np.zeros(na)
    c, h_, b, l, u = np.zeros(n), np.zeros(m1), np.zeros(m2), np.zeros(n), np.zeros(n)
    c0 = np.zeros(1)
    lib.ref_mps_fill(h, abi.i64ptr(g_off), abi.i64ptr(g_col), abi.dptr(g_val), abi.i64ptr(a_off),
                     abi.i64ptr(a_col), abi.dptr(a_val), abi.dptr(c), abi.dptr(h_), abi.dptr(b),
                     abi.dptr(l), abi.dptr(u), abi.dptr(c0))
    lib.ref_mps_free(h)
    return GeneralFormLp(CsrMatrix(m1, n, g_off, g_col, g_val), CsrMatrix(m2, n, a_off, a_col, a_val),
                         c, h_, b, l, u, float(c0[0]))
