"""B200-native restarted PDHG (cuPDLP, arXiv 2311.12180) behind the C-ABI of
include/pdlp_b200.h. The product is libpdlp_b200.so (CUDA, sm_100a); this
package is its Python mirror of the reference's API (pdhglp::solve and types).
"""
from .lp import (
    CsrMatrix,
    GeneralFormLp,
    InfeasibilityCertificate,
    Mode,
    PrimalDualPoint,
    ReducedCosts,
    RestartCriterion,
    ScalingMode,
    SolveResult,
    SolverParams,
    SolveStatus,
)
from .api import (PdlpError, ShardGroup, ShardRank, Solver, device_count, load_library, parse_mps, plan_exchange,
                  plan_shards, read_mps, solve, solve_distributed, write_solution)

__all__ = [
    "CsrMatrix",
    "GeneralFormLp",
    "InfeasibilityCertificate",
    "Mode",
    "PrimalDualPoint",
    "ReducedCosts",
    "RestartCriterion",
    "ScalingMode",
    "SolveResult",
    "SolverParams",
    "SolveStatus",
    "PdlpError",
    "Solver",
    "load_library",
    "solve",
    "read_mps",
    "parse_mps",
    "write_solution",
    "ShardGroup",
    "ShardRank",
    "device_count",
    "plan_shards",
    "plan_exchange",
    "solve_distributed",
]
