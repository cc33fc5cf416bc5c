"""Shared test helpers: golden instances and comparison utilities."""
from __future__ import annotations

import hashlib
import json
from pathlib import Path

import numpy as np

from paper_2311_12180_b200.lp import CsrMatrix, GeneralFormLp

GOLDEN = Path(__file__).resolve().parent / "golden"


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def lp_hash(lp: GeneralFormLp) -> str:
    G, A = lp.inequality_matrix, lp.equality_matrix
    return sha(G.row_offsets, G.col_indices.astype(np.int64), G.values, A.row_offsets,
               A.col_indices.astype(np.int64), A.values, lp.objective, lp.inequality_rhs,
               lp.equality_rhs, lp.lower, lp.upper, np.array([lp.objective_constant]))


def load_golden_lp(name: str) -> GeneralFormLp:
    z = np.load(GOLDEN / "suite" / f"{name}.npz")
    n = z["c"].size
    G = CsrMatrix(z["g_off"].size - 1, n, z["g_off"], z["g_col"], z["g_val"])
    A = CsrMatrix(z["a_off"].size - 1, n, z["a_off"], z["a_col"], z["a_val"])
    return GeneralFormLp(G, A, z["c"], z["h"], z["b"], z["l"], z["u"], float(z["c0"][0]))


def suite_names() -> list[str]:
    return sorted(p.stem for p in (GOLDEN / "suite").glob("*.npz"))


def ref_suite() -> dict:
    return json.loads((GOLDEN / "ref_suite.json").read_text())


def ref_c1() -> dict:
    return json.loads((GOLDEN / "ref_c1.json").read_text())


def stacked_k(lp: GeneralFormLp) -> CsrMatrix:
    """vstack(G, A) (sparse_matrix.hpp:181-200) on the host."""
    G, A = lp.inequality_matrix, lp.equality_matrix
    return CsrMatrix(lp.num_constraints, lp.num_variables,
                     np.concatenate([G.row_offsets, A.row_offsets[1:] + G.nnz]),
                     np.concatenate([G.col_indices.astype(np.int64), A.col_indices.astype(np.int64)]),
                     np.concatenate([G.values, A.values]))


def rel_err(a, b) -> float:
    a, b = np.asarray(a), np.asarray(b)
    if a.size == 0:
        return 0.0
    return float(np.max(np.abs(a - b)) / max(1.0, float(np.max(np.abs(b)))))
