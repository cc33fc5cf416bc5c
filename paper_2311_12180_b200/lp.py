"""Instance and parameter types mirroring the reference's C++ API.

  CsrMatrix      <- pdhglp::CsrMatrix        sparse_matrix.hpp:35-115
  GeneralFormLp  <- pdhglp::GeneralFormLp    lp_model.hpp:24-72
  SolverParams   <- pdhglp::SolverParams     solver.hpp:59-94
  ScalingMode    <- pdhglp::ScalingMode      scaling.hpp:16
  SolveStatus    <- pdhglp::SolveStatus      solver.hpp:26-45

Host-side containers only (numpy); the solve itself runs on the GPU through
the C-ABI (api.py). Invalid input raises ValueError, the Python counterpart of
the reference's std::invalid_argument.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field

import numpy as np

from . import abi


class SolveStatus(enum.IntEnum):
    OPTIMAL = 0
    PRIMAL_INFEASIBLE = 1
    DUAL_INFEASIBLE = 2
    ITERATION_LIMIT = 3
    TIME_LIMIT = 4
    NUMERICAL_ERROR = 5

    def __str__(self) -> str:  # to_string(SolveStatus), solver.hpp:35-45
        return abi.STATUS_NAMES[int(self)]


class RestartCriterion(enum.IntEnum):
    NONE = 0
    SUFFICIENT_DECAY = 1
    NECESSARY_DECAY = 2
    LONG_INNER_LOOP = 3

    def __str__(self) -> str:
        return abi.RESTART_NAMES[int(self)]


class ScalingMode(enum.IntEnum):
    NONE = 0
    RUIZ = 1
    RUIZ_POCK_CHAMBOLLE = 2


class Mode(enum.IntEnum):
    FAST = abi.MODE_FAST
    PARITY = abi.MODE_PARITY


@dataclass
class CsrMatrix:
    """Compressed sparse rows, int64 indices like the reference's index_t."""

    num_rows: int
    num_cols: int
    row_offsets: np.ndarray
    col_indices: np.ndarray
    values: np.ndarray

    def __post_init__(self) -> None:
        self.row_offsets = np.ascontiguousarray(self.row_offsets, dtype=np.int64)
        ci = np.asarray(self.col_indices)
        self.col_indices = np.ascontiguousarray(ci, dtype=np.int32 if ci.dtype == np.int32 else np.int64)
        self.values = np.ascontiguousarray(self.values, dtype=np.float64)
        if self.row_offsets.shape != (self.num_rows + 1,):
            raise ValueError("csr: row_offsets must have num_rows + 1 entries")
        if self.col_indices.shape != self.values.shape:
            raise ValueError("csr: col_indices and values differ in length")
        if self.row_offsets[0] != 0 or self.row_offsets[-1] != self.values.size:
            raise ValueError("csr: row_offsets must start at 0 and end at nnz")

    @property
    def nnz(self) -> int:
        return int(self.values.size)

    @staticmethod
    def zero(rows: int, cols: int) -> "CsrMatrix":
        return CsrMatrix(rows, cols, np.zeros(rows + 1, np.int64), np.zeros(0, np.int64), np.zeros(0))

    @staticmethod
    def identity(n: int) -> "CsrMatrix":
        return CsrMatrix(n, n, np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int64), np.ones(n))

    @staticmethod
    def from_triplets(rows: int, cols: int, r, c, v) -> "CsrMatrix":
        """CsrMatrix::from_triplets (sparse_matrix.hpp:57-108): sorted by
        (row, col), duplicates summed, exact zeros dropped; out-of-range
        entries raise ValueError naming the offending triplet."""
        r = np.asarray(r, dtype=np.int64)
        c = np.asarray(c, dtype=np.int64)
        v = np.asarray(v, dtype=np.float64)
        bad = np.nonzero((r < 0) | (r >= rows) | (c < 0) | (c >= cols))[0]
        if bad.size:
            i = int(bad[0])
            raise ValueError(
                f"triplet {i} at ({int(r[i])}, {int(c[i])}) is outside a {rows}x{cols} matrix"
            )
        order = np.lexsort((c, r))
        r, c, v = r[order], c[order], v[order]
        if r.size:
            new = np.ones(r.size, dtype=bool)
            new[1:] = (r[1:] != r[:-1]) | (c[1:] != c[:-1])
            starts = np.nonzero(new)[0]
            sums = np.add.reduceat(v, starts) if (~new).any() else v[starts]
            r, c, v = r[starts], c[starts], sums
            keep = v != 0.0
            r, c, v = r[keep], c[keep], v[keep]
        counts = np.bincount(r, minlength=rows) if r.size else np.zeros(rows, np.int64)
        off = np.zeros(rows + 1, np.int64)
        np.cumsum(counts, out=off[1:])
        return CsrMatrix(rows, cols, off, c, v)

    def to_dense(self) -> np.ndarray:
        d = np.zeros((self.num_rows, self.num_cols))
        rows = np.repeat(np.arange(self.num_rows), np.diff(self.row_offsets))
        d[rows, self.col_indices] = self.values
        return d

    def to_abi(self) -> abi.PdlpCsr:
        s = abi.PdlpCsr()
        s.num_rows, s.num_cols, s.nnz = self.num_rows, self.num_cols, self.nnz
        s.row_offsets = abi.i64ptr(self.row_offsets)
        if self.col_indices.dtype == np.int32:
            s.col_indices = None
            s.col_indices32 = abi.i32ptr(self.col_indices)
        else:
            s.col_indices = abi.i64ptr(self.col_indices)
            s.col_indices32 = None
        s.values = abi.dptr(self.values)
        return s


@dataclass
class GeneralFormLp:
    """min c'x  s.t.  Gx >= h,  Ax = b,  l <= x <= u   (lp_model.hpp:24-43)."""

    inequality_matrix: CsrMatrix
    equality_matrix: CsrMatrix
    objective: np.ndarray
    inequality_rhs: np.ndarray
    equality_rhs: np.ndarray
    lower: np.ndarray
    upper: np.ndarray
    objective_constant: float = 0.0

    def __post_init__(self) -> None:
        for name in ("objective", "inequality_rhs", "equality_rhs", "lower", "upper"):
            setattr(self, name, np.ascontiguousarray(getattr(self, name), dtype=np.float64))

    @property
    def num_variables(self) -> int:
        return int(self.objective.size)

    @property
    def num_inequalities(self) -> int:
        return self.inequality_matrix.num_rows

    @property
    def num_equalities(self) -> int:
        return self.equality_matrix.num_rows

    @property
    def num_constraints(self) -> int:
        return self.num_inequalities + self.num_equalities

    @property
    def nnz(self) -> int:
        return self.inequality_matrix.nnz + self.equality_matrix.nnz

    def validate(self) -> None:
        """GeneralFormLp::validate (lp_model.hpp:45-72), plus the CSR storage
        checks the raw-pointer C ABI needs."""
        self.validate_shapes()
        nan = np.nonzero(np.isnan(self.lower) | np.isnan(self.upper))[0]
        if nan.size:
            raise ValueError(f"lp: NaN bound on variable {int(nan[0])}")
        bad = np.nonzero((self.lower > self.upper) | (self.lower == np.inf) | (self.upper == -np.inf))[0]
        if bad.size:
            raise ValueError(f"lp: empty bound interval on variable {int(bad[0])}")
        if np.isnan(self.objective).any():
            raise ValueError("lp: NaN objective entry")

    def validate_shapes(self) -> None:
        """The array-length half of validate(): what the raw-pointer C ABI
        cannot check itself (it would read past a short array). The value
        checks (NaN and empty bounds, NaN objective) are repeated by
        pdlp_create with the same messages."""
        for name, M in (("inequality", self.inequality_matrix), ("equality", self.equality_matrix)):
            if M.row_offsets.size != M.num_rows + 1:
                raise ValueError(f"lp: {name} matrix row_offsets must have num_rows + 1 entries")
            if M.col_indices.size != M.values.size:
                raise ValueError(f"lp: {name} matrix col_indices and values differ in length")
            if M.num_rows >= 0 and (M.row_offsets[0] != 0 or M.row_offsets[-1] != M.values.size):
                raise ValueError(f"lp: {name} matrix row_offsets must run from 0 to nnz")
        n = self.num_variables
        if self.inequality_matrix.num_cols != n or self.equality_matrix.num_cols != n:
            raise ValueError("lp: constraint matrices must have n columns")
        if self.inequality_rhs.size != self.num_inequalities or self.equality_rhs.size != self.num_equalities:
            raise ValueError("lp: rhs length does not match row count")
        if self.lower.size != n or self.upper.size != n:
            raise ValueError("lp: bound vectors must have length n")

    def to_abi(self) -> abi.PdlpLp:
        s = abi.PdlpLp()
        s.inequality_matrix = self.inequality_matrix.to_abi()
        s.equality_matrix = self.equality_matrix.to_abi()
        s.num_variables = self.num_variables
        s.objective = abi.dptr(self.objective)
        s.inequality_rhs = abi.dptr(self.inequality_rhs)
        s.equality_rhs = abi.dptr(self.equality_rhs)
        s.lower = abi.dptr(self.lower)
        s.upper = abi.dptr(self.upper)
        s.objective_constant = float(self.objective_constant)
        return s


@dataclass
class SolverParams:
    """SolverParams (solver.hpp:59-77) with the same defaults, plus B200 knobs."""

    eps_optimal: float = 1e-4
    eps_infeasible: float = 1e-8
    time_limit_seconds: float = 3600.0
    iteration_limit: int = 2**63 - 1
    beta_sufficient: float = 0.2
    beta_necessary: float = 0.8
    beta_artificial: float = 0.36
    theta_smoothing: float = 0.5
    eps_zero: float = 1e-10
    evaluation_frequency: int = 64
    scaling: ScalingMode = ScalingMode.RUIZ_POCK_CHAMBOLLE
    ruiz_iterations: int = 10
    pock_chambolle_alpha: float = 1.0
    step_reduction_exponent: float = 0.3
    step_growth_exponent: float = 0.6
    omega_min: float = 1e-8
    omega_max: float = 1e8
    record_step_log: bool = False
    # B200 extensions
    device: int = 0
    mode: Mode = Mode.FAST
    use_cuda_graph: bool = True
    l2_persist: bool = False  # access-policy window on the gathered iterate (opt-in)
    engine: int = 0  # abi.ENGINE_*: AUTO = the CUDA-graph window (STREAM without graphs)
    # row sharding: rank `rank` of `world_size` (see ShardGroup)
    world_size: int = 1
    rank: int = 0
    plan_world: int = 0  # tile breaks of a plan_world-way partition on one rank (verification)

    def validate(self) -> None:
        """SolverParams::validate (solver.hpp:79-93)."""
        if not (self.eps_optimal > 0.0) or not (self.eps_infeasible > 0.0):
            raise ValueError("params: tolerances must be positive")
        if not (0.0 < self.beta_sufficient < self.beta_necessary < 1.0):
            raise ValueError("params: need 0 < beta_sufficient < beta_necessary < 1")
        if self.theta_smoothing < 0.0 or self.theta_smoothing > 1.0:
            raise ValueError("params: theta_smoothing must lie in [0, 1]")
        if self.evaluation_frequency < 1:
            raise ValueError("params: evaluation_frequency must be >= 1")

    def to_abi(self) -> abi.PdlpParams:
        p = abi.PdlpParams()
        for name, _ in abi.PdlpParams._fields_:
            if name == "reserved":
                continue
            v = getattr(self, name)
            setattr(p, name, int(v) if isinstance(v, (bool, enum.IntEnum)) else v)
        return p


class ReducedCosts:
    """ReducedCosts (lp_model.hpp:147-176): lambda and its positive / negative
    parts. The parts are formed from lambda on first use (two fewer n-vectors
    to copy out of every solve)."""

    def __init__(self, lambda_: np.ndarray, lambda_pos: np.ndarray | None = None,
                 lambda_neg: np.ndarray | None = None):
        self.lambda_ = lambda_
        self._pos, self._neg = lambda_pos, lambda_neg

    @property
    def lambda_pos(self) -> np.ndarray:
        if self._pos is None:
            self._pos = np.where(self.lambda_ > 0.0, self.lambda_, 0.0)
        return self._pos

    @property
    def lambda_neg(self) -> np.ndarray:
        if self._neg is None:
            self._neg = np.where(self.lambda_ < 0.0, -self.lambda_, 0.0)
        return self._neg

    def __repr__(self) -> str:
        return f"ReducedCosts(n={len(self.lambda_)})"


@dataclass
class PrimalDualPoint:
    primal: np.ndarray
    dual: np.ndarray


@dataclass
class InfeasibilityCertificate:
    status: SolveStatus
    primal_ray: np.ndarray | None = None
    dual_ray: np.ndarray | None = None
    dual_ray_reduced_costs: ReducedCosts | None = None


@dataclass
class SolveResult:
    """SolveResult (solver.hpp:618-630)."""

    status: SolveStatus
    point: PrimalDualPoint
    reduced: ReducedCosts
    info: dict
    iterations: int
    restarts: int
    solve_seconds: float
    certificate: InfeasibilityCertificate | None = None
    step_log: np.ndarray = field(default_factory=lambda: np.zeros(0, abi.STEP_LOG_DTYPE))
    restart_log: np.ndarray = field(default_factory=lambda: np.zeros(0, abi.RESTART_DTYPE))
    message: str = ""


def result_from_buffers(info: abi.PdlpResultInfo, x, y, lam, pos, neg, step_log, restart_log) -> SolveResult:
    d = abi.info_to_dict(info)
    status = SolveStatus(info.status)
    cert = None
    red = ReducedCosts(lam, pos, neg)
    if info.has_certificate:
        if status == SolveStatus.PRIMAL_INFEASIBLE:
            cert = InfeasibilityCertificate(status, dual_ray=y.copy(), dual_ray_reduced_costs=red)
        else:
            cert = InfeasibilityCertificate(status, primal_ray=x.copy())
    return SolveResult(
        status=status,
        point=PrimalDualPoint(x, y),
        reduced=red,
        info=d,
        iterations=int(info.iterations),
        restarts=int(info.restarts),
        solve_seconds=float(info.solve_seconds),
        certificate=cert,
        step_log=step_log,
        restart_log=restart_log,
        message=d["message"],
    )


__all__ = [
    "CsrMatrix",
    "GeneralFormLp",
    "SolverParams",
    "SolveStatus",
    "RestartCriterion",
    "ScalingMode",
    "Mode",
    "ReducedCosts",
    "PrimalDualPoint",
    "InfeasibilityCertificate",
    "SolveResult",
    "result_from_buffers",
    "C",
]
