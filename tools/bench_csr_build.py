"""GPU CsrMatrix::from_triplets at scale: time
pdlp_csr_from_triplets (host triplets in, host CSR out, copies included) on
seeded C4/C5-shaped triplet sets and check the integer output exactly.

  python tools/bench_csr_build.py 200 500     # millions of triplets

Per size: rows = nnz / 10, cols = nnz / 5 (the C4 recipe's shape), triplets in
random order without duplicates. Checks: row_offsets == cumsum(bincount(rows));
the output keys (row * cols + col) strictly increasing and equal to the sorted
input keys; values are the input values of those keys. The reference's host
from_triplets takes 1.19 s at 20 M.
"""
from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2311_12180_b200.api import csr_from_triplets  # noqa: E402


def run(millions: int) -> dict:
    nt = millions * 1_000_000
    rows, cols = nt // 10, nt // 5
    rng = np.random.default_rng(20261004 + millions)
    t = time.perf_counter()
    # distinct keys without a set: a random permutation of a strided key range
    keys = np.arange(nt, dtype=np.int64) * ((rows * cols) // nt)
    keys += rng.integers(0, (rows * cols) // nt, nt)
    rng.shuffle(keys)
    r, c = keys // cols, keys % cols
    v = rng.uniform(-3.0, 3.0, nt)
    gen_s = time.perf_counter() - t
    t = time.perf_counter()
    g = csr_from_triplets(rows, cols, r, c, v)
    build_s = time.perf_counter() - t
    ok_off = bool(np.array_equal(g.row_offsets, np.concatenate([[0], np.cumsum(np.bincount(r, minlength=rows))])))
    out_rows = np.repeat(np.arange(rows, dtype=np.int64), np.diff(g.row_offsets))
    out_keys = out_rows * cols + g.col_indices
    ok_inc = bool(np.all(np.diff(out_keys) > 0))
    order = np.argsort(keys, kind="stable")
    ok_keys = bool(np.array_equal(out_keys, keys[order]))
    ok_vals = bool(np.array_equal(g.values, v[order]))
    return {"triplets": nt, "rows": rows, "cols": cols, "generate_s": gen_s, "gpu_from_triplets_s": build_s,
            "triplets_per_s": nt / build_s, "offsets_exact": ok_off, "keys_strictly_increasing": ok_inc,
            "keys_exact": ok_keys, "values_exact": ok_vals}


if __name__ == "__main__":
    for mm in [int(a) for a in sys.argv[1:]] or [20]:
        print(json.dumps(run(mm)), flush=True)
