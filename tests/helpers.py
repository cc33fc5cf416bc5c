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


def write_free_mps(lp: GeneralFormLp, path, name: str = "LP") -> None:
    """Writes `lp` as free-format MPS that read_mps parses back to the same
    GeneralFormLp (inequality rows as G rows first, then E rows; values with
    17 significant digits; the objective constant as -RHS of the N row,
    mps_io.hpp:403,508). Test helper: turns the golden .npz instances back
    into files for the directory benchmark."""
    G, A = lp.inequality_matrix, lp.equality_matrix
    n, m1, m2 = lp.num_variables, G.num_rows, A.num_rows
    f = lambda v: repr(float(v))  # noqa: E731  (shortest round-trip repr)
    cols: list[list[tuple[str, float]]] = [[] for _ in range(n)]
    for mat, prefix in ((G, "G"), (A, "E")):
        for r in range(mat.num_rows):
            for k in range(int(mat.row_offsets[r]), int(mat.row_offsets[r + 1])):
                cols[int(mat.col_indices[k])].append((f"{prefix}{r}", float(mat.values[k])))
    out = [f"NAME {name}", "ROWS", " N OBJ"]
    out += [f" G G{r}" for r in range(m1)] + [f" E E{r}" for r in range(m2)]
    out.append("COLUMNS")
    for j in range(n):
        out.append(f" X{j} OBJ {f(lp.objective[j])}")
        out += [f" X{j} {row} {f(v)}" for row, v in cols[j]]
    out.append("RHS")
    if lp.objective_constant != 0.0:
        out.append(f" RHS OBJ {f(-lp.objective_constant)}")
    out += [f" RHS G{r} {f(v)}" for r, v in enumerate(lp.inequality_rhs) if v != 0.0]
    out += [f" RHS E{r} {f(v)}" for r, v in enumerate(lp.equality_rhs) if v != 0.0]
    out.append("BOUNDS")
    inf = float("inf")
    for j, (lo, up) in enumerate(zip(lp.lower, lp.upper)):
        if lo == up:
            out.append(f" FX BND X{j} {f(lo)}")
            continue
        if lo == -inf and up == inf:
            out.append(f" FR BND X{j}")
            continue
        if lo == -inf:
            out.append(f" MI BND X{j}")
        elif lo != 0.0:
            out.append(f" LO BND X{j} {f(lo)}")
        if up != inf:
            out.append(f" UP BND X{j} {f(up)}")
    out.append("ENDATA")
    Path(path).write_text("\n".join(out) + "\n")
