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

# PDLP_LIB selects an A/B build variant of the same library (tools/build_variants.py)
_LIB_PATH = Path(os.environ.get("PDLP_LIB") or Path(__file__).resolve().parent / "lib" / "libpdlp_b200.so")
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
        "pdlp_device_count": (C.c_int, [i32p]),
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
        "pdlp_kernel_bytes": (C.c_int, [H, C.c_int32, dp]),
        "pdlp_get_sizes": (C.c_int, [H, i64p]),
        "pdlp_last_error": (C.c_char_p, []),
        "pdlp_read_mps": (C.c_int, [C.c_char_p, C.c_int32, C.POINTER(H)]),
        "pdlp_parse_mps": (C.c_int, [C.c_char_p, C.c_int64, C.c_int32, C.POINTER(H)]),
        "pdlp_lp_file_lp": (C.POINTER(abi.PdlpLp), [H]),
        "pdlp_lp_file_name": (C.c_char_p, [H]),
        "pdlp_lp_file_column_name": (C.c_char_p, [H, C.c_int64]),
        "pdlp_lp_file_free": (None, [H]),
        "pdlp_write_solution": (C.c_int, [C.c_char_p, C.POINTER(abi.PdlpResultInfo), dp, C.c_int64, dp,
                                          C.c_int64]),
        "pdlp_csr_from_triplets": (C.c_int, [C.c_int64, C.c_int64, C.c_int64, i64p, i64p, dp, C.c_int32, i64p,
                                             i64p, dp, i64p]),
        "pdlp_shard_blob_size": (C.c_int64, []),
        "pdlp_shard_link_local": (C.c_int, [C.POINTER(H), C.c_int32]),
        "pdlp_shard_export": (C.c_int, [H, C.c_void_p, C.c_int64]),
        "pdlp_shard_import": (C.c_int, [H, C.c_void_p, C.c_int32]),
        "pdlp_shard_info": (C.c_int, [H, i64p]),
        "pdlp_shard_exchange": (C.c_int, [H, i64p]),
        "pdlp_pdhg_raw_step": (C.c_int, [H, dp, dp, C.c_double, C.c_double, dp, dp]),
        "pdlp_plan_shards": (C.c_int, [C.POINTER(abi.PdlpLp), C.c_int32, i64p, i64p]),
        "pdlp_plan_exchange": (C.c_int, [C.POINTER(abi.PdlpLp), C.c_int32, i64p, i64p, C.c_void_p, C.c_void_p]),
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
        lp.validate_shapes()  # the C ABI reads the arrays through raw pointers (it checks the values itself)
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
        x, y, lam = np.empty(n), np.empty(m), np.empty(n)
        _check(self._lib.pdlp_get_solution(self._h, abi.dptr(x), abi.dptr(y), abi.dptr(lam), None, None))
        pos = neg = None  # formed from lambda on first use (ReducedCosts)
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
        transpose = op in (abi.OP_KT_SCALED, abi.OP_KT_ORIGINAL)
        if v.ndim != 1 or v.size != (self.m if transpose else self.n):
            raise ValueError("spmv: dimension mismatch")  # sparse_matrix.hpp:119-122,144-147
        out = np.zeros(self.n if transpose else self.m)
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

    def pdhg_raw_step(self, x, y, tau: float, sigma: float) -> tuple[np.ndarray, np.ndarray]:
        """pdhg_raw_step (solver.hpp:335-358) on the unscaled saddle problem:
        one plain PDHG step from (x, y), returning (x', y')."""
        n, m = self.n, self.m
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.ascontiguousarray(y, dtype=np.float64)
        if x.size != n or y.size != m:
            raise ValueError("pdhg_raw_step: dimension mismatch")
        xo, yo = np.empty(n), np.empty(m)
        _check(self._lib.pdlp_pdhg_raw_step(self._h, abi.dptr(x), abi.dptr(y), float(tau), float(sigma),
                                            abi.dptr(xo), abi.dptr(yo)))
        return xo, yo

    # ---- row sharding ----
    def shard_info(self) -> dict:
        out = np.zeros(10, np.int64)
        _check(self._lib.pdlp_shard_info(self._h, abi.i64ptr(out)))
        keys = ("world", "rank", "row0", "row1", "col0", "col1", "k_tiles", "kt_tiles", "k_tiles_all",
                "kt_tiles_all")
        return {k: int(v) for k, v in zip(keys, out)}

    def shard_exchange(self) -> dict:
        """Values this rank pushes to peers per trial (with the gather masks,
        and with an all-to-all push) and the nonzeros of K and K^T it stores
        (pdlp_shard_exchange)."""
        out = np.zeros(4, np.int64)
        _check(self._lib.pdlp_shard_exchange(self._h, abi.i64ptr(out)))
        return {"pushed": int(out[0]), "all_to_all": int(out[1]), "k_nnz": int(out[2]), "kt_nnz": int(out[3])}

    def shard_export(self) -> bytes:
        size = int(self._lib.pdlp_shard_blob_size())
        buf = C.create_string_buffer(size)
        _check(self._lib.pdlp_shard_export(self._h, buf, size))
        return buf.raw

    def shard_import(self, blobs: list[bytes]) -> None:
        data = b"".join(blobs)
        _check(self._lib.pdlp_shard_import(self._h, data, len(blobs)))

    def time_kernel(self, which: int, reps: int = 50) -> tuple[float, float]:
        ms, by = C.c_double(), C.c_double()
        _check(self._lib.pdlp_time_kernel(self._h, which, reps, C.byref(ms), C.byref(by)))
        return ms.value, by.value

    def kernel_bytes(self, which: int) -> dict:
        """Algorithmic and moved bytes of one launch of kernel
        `which` (0 dual, 1 primal, 2 K x, 3 K^T y), and the panel count."""
        out = (C.c_double * 3)()
        _check(self._lib.pdlp_kernel_bytes(self._h, which, out))
        return {"algorithmic": out[0], "moved": out[1], "panels": int(out[2])}


def csr_from_triplets(rows: int, cols: int, r, c, v, device: int = 0):
    """CsrMatrix::from_triplets (sparse_matrix.hpp:57-108) on the GPU."""
    from .lp import CsrMatrix

    lib = load_library()
    r = np.ascontiguousarray(r, dtype=np.int64)
    c = np.ascontiguousarray(c, dtype=np.int64)
    v = np.ascontiguousarray(v, dtype=np.float64)
    off, col, val = np.zeros(rows + 1, np.int64), np.zeros(r.size, np.int64), np.zeros(r.size)
    nnz = C.c_int64()
    _check(lib.pdlp_csr_from_triplets(rows, cols, r.size, abi.i64ptr(r), abi.i64ptr(c), abi.dptr(v), device,
                                      abi.i64ptr(off), abi.i64ptr(col), abi.dptr(val), C.byref(nnz)))
    k = nnz.value
    return CsrMatrix(rows, cols, off, col[:k].copy(), val[:k].copy())


def plan_shards(lp: GeneralFormLp, world: int) -> tuple[np.ndarray, np.ndarray]:
    """Row cuts (world + 1 each) of K = (G; A) and of K^T a world-way sharded
    solve uses; host-only (no device)."""
    lib = load_library()
    kc, ktc = np.zeros(world + 1, np.int64), np.zeros(world + 1, np.int64)
    lpa = lp.to_abi()
    _check(lib.pdlp_plan_shards(C.byref(lpa), world, abi.i64ptr(kc), abi.i64ptr(ktc)))
    return kc, ktc


def plan_exchange(lp: GeneralFormLp, world: int) -> dict:
    """Gather masks and per-rank exchange volumes of a world-way sharded solve
    (pdlp_plan_exchange; host only, no GPU): xmask (n) / ymask (m) as uint32
    bit sets of the ranks that gather each x' / y' value, and per rank the
    values pushed per trial with the masks and with an all-to-all push."""
    lib = load_library()
    lpa = lp.to_abi()
    pushed, a2a = np.zeros(world, np.int64), np.zeros(world, np.int64)
    xm, ym = np.zeros(lp.num_variables, np.uint32), np.zeros(lp.num_constraints, np.uint32)
    _check(lib.pdlp_plan_exchange(C.byref(lpa), world, abi.i64ptr(pushed), abi.i64ptr(a2a),
                                  xm.ctypes.data_as(C.c_void_p), ym.ctypes.data_as(C.c_void_p)))
    return {"pushed": pushed, "all_to_all": a2a, "xmask": xm, "ymask": ym}


class ShardGroup:
    """All ranks of one row-sharded solve inside this process (the loopback
    transport: every rank gets its own stream and buffers, usually on one
    device; the ranks' kernels write each other's buffers exactly as they write
    peer GPUs' memory over NVLink). solve() runs the ranks in one host thread
    each, like one process per GPU would; every rank returns the same result."""

    def __init__(self, lp: GeneralFormLp, params: SolverParams | None, world: int, devices=None):
        import dataclasses

        base = params or SolverParams()
        self.ranks = []
        for q in range(world):
            dev = base.device if devices is None else devices[q]
            p = dataclasses.replace(base, world_size=world, rank=q, device=dev)
            self.ranks.append(Solver(lp, p))
        arr = (C.c_void_p * world)(*[r._h for r in self.ranks])
        _check(self.ranks[0]._lib.pdlp_shard_link_local(arr, world))

    def solve(self) -> list[SolveResult]:
        import threading

        out: list = [None] * len(self.ranks)

        def run(q):
            try:
                out[q] = self.ranks[q].solve()
            except BaseException as e:  # noqa: BLE001 - re-raised below
                out[q] = e

        ts = [threading.Thread(target=run, args=(q,)) for q in range(len(self.ranks))]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        for r in out:
            if isinstance(r, BaseException):
                raise r
        return out

    def close(self) -> None:
        for r in self.ranks:
            r.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


class ShardRank:
    """One rank of a row-sharded solve, one process per GPU: the
    rank and world come from torch.distributed (any backend; only the ~1 KB
    CUDA-IPC blobs travel over it), the device from LOCAL_RANK (modulo the
    visible devices, so a one-GPU box can host several ranks for tests).
    After the blob exchange the ranks move data GPU-to-GPU inside the kernels
    (csrc/shard.cuh). The handle stays linked for repeated solves."""

    def __init__(self, lp: GeneralFormLp, params: SolverParams | None = None, group=None, device=None):
        import dataclasses

        import torch.distributed as dist

        world, rank = dist.get_world_size(group), dist.get_rank(group)
        if device is None:
            device = int(os.environ.get("LOCAL_RANK", rank)) % max(1, device_count())
        base = params or SolverParams()
        self.rank, self.world, self.device = rank, world, device
        self.solver = Solver(lp, dataclasses.replace(base, world_size=world, rank=rank, device=device))
        try:
            blobs: list = [None] * world
            dist.all_gather_object(blobs, self.solver.shard_export(), group=group)
            self.solver.shard_import(blobs)
            dist.barrier(group)
        except BaseException:
            self.solver.close()
            raise

    def solve(self) -> SolveResult:
        return self.solver.solve()

    def close(self) -> None:
        self.solver.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def solve_distributed(lp: GeneralFormLp, params: SolverParams | None = None, group=None, device=None) -> SolveResult:
    """One rank of a row-sharded solve, one process per GPU (ShardRank): every
    rank returns the same result."""
    with ShardRank(lp, params, group, device) as r:
        return r.solve()


MPS_FIXED, MPS_FREE, MPS_AUTO = 0, 1, 2


def _lp_from_file(lib, h) -> GeneralFormLp:
    from .lp import CsrMatrix

    v = lib.pdlp_lp_file_lp(h).contents

    def csr(c):
        rows, nnz = int(c.num_rows), int(c.nnz)
        off = np.ctypeslib.as_array(c.row_offsets, (rows + 1,)).copy()
        col = np.ctypeslib.as_array(c.col_indices, (nnz,)).copy() if nnz else np.zeros(0, np.int64)
        val = np.ctypeslib.as_array(c.values, (nnz,)).copy() if nnz else np.zeros(0)
        return CsrMatrix(rows, int(c.num_cols), off, col, val)

    n = int(v.num_variables)
    m1, m2 = int(v.inequality_matrix.num_rows), int(v.equality_matrix.num_rows)

    def vec(p, k):
        return np.ctypeslib.as_array(p, (k,)).copy() if k else np.zeros(0)

    return GeneralFormLp(csr(v.inequality_matrix), csr(v.equality_matrix), vec(v.objective, n),
                         vec(v.inequality_rhs, m1), vec(v.equality_rhs, m2), vec(v.lower, n), vec(v.upper, n),
                         float(v.objective_constant))


def device_count() -> int:
    """Visible CUDA devices (pdlp_device_count)."""
    n = C.c_int32(0)
    _check(load_library().pdlp_device_count(C.byref(n)))
    return int(n.value)


def read_mps(path, fmt: int = MPS_AUTO) -> GeneralFormLp:
    """read_mps_file (mps_io.hpp:582-585), host C++ in libpdlp_b200.so. Parse
    errors raise PdlpError naming the line; crossing bounds raise ValueError."""
    lib = load_library()
    h = C.c_void_p()
    _check(lib.pdlp_read_mps(str(path).encode(), fmt, C.byref(h)))
    try:
        return _lp_from_file(lib, h)
    finally:
        lib.pdlp_lp_file_free(h)


def parse_mps(text: str, fmt: int = MPS_AUTO) -> GeneralFormLp:
    """parse_mps + to_general_form (mps_io.hpp:163-554) on in-memory text."""
    lib = load_library()
    b = text.encode()
    h = C.c_void_p()
    _check(lib.pdlp_parse_mps(b, len(b), fmt, C.byref(h)))
    try:
        return _lp_from_file(lib, h)
    finally:
        lib.pdlp_lp_file_free(h)


def write_solution(result: SolveResult, path, include_vectors: bool = False) -> None:
    """write_solution (solution_io.hpp:70-95)."""
    lib = load_library()
    info = abi.PdlpResultInfo()
    info.status = int(result.status)
    for k in ("primal_objective", "dual_objective", "relative_gap", "primal_residual_norm",
              "dual_residual_norm"):
        setattr(info, k, float(result.info[k]))
    info.iterations = int(result.iterations)
    info.solve_seconds = float(result.solve_seconds)
    x = np.ascontiguousarray(result.point.primal, dtype=np.float64)
    y = np.ascontiguousarray(result.point.dual, dtype=np.float64)
    _check(lib.pdlp_write_solution(str(path).encode(), C.byref(info), abi.dptr(x) if include_vectors else None,
                                   x.size, abi.dptr(y) if include_vectors else None, y.size))


def solve(lp: GeneralFormLp, params: SolverParams | None = None) -> SolveResult:
    """pdhglp::solve (solver.hpp:935-940) on the GPU."""
    lp.validate()
    (params or SolverParams()).validate()
    with Solver(lp, params) as s:
        return s.solve()


__all__ = ["Solver", "ShardRank", "plan_exchange", "solve", "load_library", "default_params", "PdlpError", "library_path", "read_mps",
           "parse_mps", "write_solution", "MPS_FIXED", "MPS_FREE", "MPS_AUTO", "ShardGroup", "plan_shards",
           "csr_from_triplets",
           "solve_distributed"]
