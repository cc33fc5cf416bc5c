"""ctypes mirror of the C-ABI structs in include/pdlp_b200.h.

One description serves the GPU library (libpdlp_b200.so), and — in tests and
the bench's CPU arm only — the CPU checkers under oracle/.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

PDLP_OK, PDLP_EINVAL, PDLP_ERUNTIME, PDLP_ECUDA, PDLP_ESTATE = 0, 1, 2, 3, 4

STATUS_NAMES = [
    "optimal",
    "primal_infeasible",
    "dual_infeasible",
    "iteration_limit",
    "time_limit",
    "numerical_error",
    "running",
]

RESTART_NAMES = ["none", "sufficient_decay", "necessary_decay_no_progress", "long_inner_loop"]

OP_K_SCALED, OP_KT_SCALED, OP_K_ORIGINAL, OP_KT_ORIGINAL = 0, 1, 2, 3
MODE_FAST, MODE_PARITY = 0, 1
ENGINE_AUTO, ENGINE_PERSISTENT, ENGINE_GRAPH, ENGINE_STREAM = 0, 1, 2, 3

_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)
_i32p = C.POINTER(C.c_int32)


class PdlpCsr(C.Structure):
    _fields_ = [
        ("num_rows", C.c_int64),
        ("num_cols", C.c_int64),
        ("nnz", C.c_int64),
        ("row_offsets", _i64p),
        ("col_indices", _i64p),
        ("col_indices32", _i32p),
        ("values", _dp),
    ]


class PdlpStandardOptions(C.Structure):
    """pdlp_standard_options (StandardPdhgOptions, standard_form.hpp:100-113)."""

    _fields_ = [
        ("step_size", C.c_double),
        ("restart_decay", C.c_double),
        ("convergence_tol", C.c_double),
        ("iteration_limit", C.c_int64),
        ("parity", C.c_int32),
        ("device", C.c_int32),
        ("reserved", C.c_int64 * 4),
    ]


class PdlpLp(C.Structure):
    _fields_ = [
        ("inequality_matrix", PdlpCsr),
        ("equality_matrix", PdlpCsr),
        ("num_variables", C.c_int64),
        ("objective", _dp),
        ("inequality_rhs", _dp),
        ("equality_rhs", _dp),
        ("lower", _dp),
        ("upper", _dp),
        ("objective_constant", C.c_double),
    ]


class PdlpParams(C.Structure):
    _fields_ = [
        ("eps_optimal", C.c_double),
        ("eps_infeasible", C.c_double),
        ("time_limit_seconds", C.c_double),
        ("iteration_limit", C.c_int64),
        ("beta_sufficient", C.c_double),
        ("beta_necessary", C.c_double),
        ("beta_artificial", C.c_double),
        ("theta_smoothing", C.c_double),
        ("eps_zero", C.c_double),
        ("evaluation_frequency", C.c_int64),
        ("scaling", C.c_int32),
        ("ruiz_iterations", C.c_int32),
        ("pock_chambolle_alpha", C.c_double),
        ("step_reduction_exponent", C.c_double),
        ("step_growth_exponent", C.c_double),
        ("omega_min", C.c_double),
        ("omega_max", C.c_double),
        ("record_step_log", C.c_int32),
        ("device", C.c_int32),
        ("mode", C.c_int32),
        ("use_cuda_graph", C.c_int32),
        ("l2_persist", C.c_int32),
        ("engine", C.c_int32),
        ("world_size", C.c_int32),
        ("rank", C.c_int32),
        ("plan_world", C.c_int32),
        ("reserved", C.c_int32 * 3),
    ]


class PdlpResultInfo(C.Structure):
    _fields_ = [
        ("status", C.c_int32),
        ("has_certificate", C.c_int32),
        ("iterations", C.c_int64),
        ("restarts", C.c_int64),
        ("solve_seconds", C.c_double),
        ("setup_seconds", C.c_double),
        ("device_seconds", C.c_double),
        ("window_seconds", C.c_double),
        ("primal_objective", C.c_double),
        ("dual_objective", C.c_double),
        ("primal_objective_raw", C.c_double),
        ("dual_objective_raw", C.c_double),
        ("gap_abs", C.c_double),
        ("primal_residual_norm", C.c_double),
        ("dual_residual_norm", C.c_double),
        ("relative_gap", C.c_double),
        ("relative_primal_residual", C.c_double),
        ("relative_dual_residual", C.c_double),
        ("kkt_omega", C.c_double),
        ("step_log_size", C.c_int64),
        ("restart_log_size", C.c_int64),
        ("num_variables", C.c_int64),
        ("num_constraints", C.c_int64),
        ("trials", C.c_int64),
        ("evaluations", C.c_int64),
        ("gpu_launches", C.c_int64),
        ("eval_seconds", C.c_double),
        ("message", C.c_char * 256),
    ]


class PdlpStepLogEntry(C.Structure):
    _fields_ = [
        ("step_counter", C.c_int64),
        ("omega", C.c_double),
        ("eta_accepted", C.c_double),
        ("eta_bar", C.c_double),
        ("eta_next", C.c_double),
        ("movement_sq", C.c_double),
        ("interaction", C.c_double),
    ]


class PdlpRestartEvent(C.Structure):
    _fields_ = [
        ("total_iterations", C.c_int64),
        ("epoch_length", C.c_int64),
        ("criterion", C.c_int32),
        ("candidate_is_average", C.c_int32),
        ("kkt_candidate", C.c_double),
        ("kkt_previous_candidate", C.c_double),
        ("kkt_epoch_start", C.c_double),
        ("omega_before", C.c_double),
        ("omega_after", C.c_double),
    ]


STEP_LOG_DTYPE = np.dtype(
    [
        ("step_counter", np.int64),
        ("omega", np.float64),
        ("eta_accepted", np.float64),
        ("eta_bar", np.float64),
        ("eta_next", np.float64),
        ("movement_sq", np.float64),
        ("interaction", np.float64),
    ]
)
RESTART_DTYPE = np.dtype(
    [
        ("total_iterations", np.int64),
        ("epoch_length", np.int64),
        ("criterion", np.int32),
        ("candidate_is_average", np.int32),
        ("kkt_candidate", np.float64),
        ("kkt_previous_candidate", np.float64),
        ("kkt_epoch_start", np.float64),
        ("omega_before", np.float64),
        ("omega_after", np.float64),
    ]
)
assert STEP_LOG_DTYPE.itemsize == C.sizeof(PdlpStepLogEntry)
assert RESTART_DTYPE.itemsize == C.sizeof(PdlpRestartEvent)


def dptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def i64ptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.int64 and a.flags.c_contiguous
    return a.ctypes.data_as(_i64p)


def i32ptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.int32 and a.flags.c_contiguous
    return a.ctypes.data_as(_i32p)


def info_to_dict(info: PdlpResultInfo) -> dict:
    d = {name: getattr(info, name) for name, _ in PdlpResultInfo._fields_ if name != "message"}
    d["message"] = info.message.decode(errors="replace")
    d["status_name"] = STATUS_NAMES[info.status] if 0 <= info.status < len(STATUS_NAMES) else "unknown"
    return d
