"""Regenerates tests/golden/standard_golden.npz from the REFERENCE's
standard-form theory harness (pdhglp/standard_form.hpp through oracle/_ref,
built from /root/reference by oracle/Makefile). Run in the build container:

    make -C oracle ref && python tests/golden/make_golden_standard.py

Instances: the five fixtures of test_standard_form.cpp / acceptance criterion
5 (acceptance_main.cpp:236-253) and two seeded random feasible standard-form
LPs (x0 >= 0, b = A x0; c = A'y0 + s0 with s0 >= 0). Per instance, arrays
prefixed "<name>/": the CSR, b, c; spectral_norm(A, 1e-12, 100000); the trace
of restarted_pdhg_standard with s = 0.9 / (2 ||A||), beta 0.5 (epoch start
KKT values, lengths, counters, last epoch start, first recorded iterates);
kkt_error_standard and p_s_norm_squared at seeded random points. Plus the
already-optimal restart chain of test_standard_form.cpp:112-127, and a
numerical-failure run (f4 with step 1e150).
"""
from __future__ import annotations

import ctypes as C
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import oracle as O  # noqa: E402
from paper_2311_12180_b200 import abi  # noqa: E402

OUT = Path(__file__).resolve().parent / "standard_golden.npz"
REC = 200  # recorded iterates kept per instance


def csr(m, n, trip):
    trip = sorted(trip)
    off = np.zeros(m + 1, np.int64)
    for r, _, _ in trip:
        off[r + 1] += 1
    return np.cumsum(off).astype(np.int64), np.array([t[1] for t in trip], np.int64), \
        np.array([t[2] for t in trip], np.float64)


def fixtures():
    out = {
        "f0": (1, 1, [(0, 0, 1.0)], [1.0], [1.0]),
        "f1": (1, 2, [(0, 0, 1.0), (0, 1, 1.0)], [1.0], [1.0, 2.0]),
        "f2": (2, 2, [(0, 0, 1.0), (1, 1, 1.0)], [1.0, 2.0], [1.0, 1.0]),
        "f3": (2, 3, [(0, 0, 1.0), (0, 1, 1.0), (1, 1, 1.0), (1, 2, 1.0)], [1.0, 1.0], [1.0, 1.0, 1.0]),
        "f4": (3, 5, [(0, 0, 1.0), (0, 2, 1.0), (0, 3, 0.5), (1, 1, 1.0), (1, 2, -1.0), (2, 3, 1.0), (2, 4, 1.0)],
               [2.0, 0.5, 1.5], [1.0, 2.0, 0.5, 1.0, 3.0]),
    }
    for name, (m, n, per_col, seed) in {"r30x60": (30, 60, 3, 5), "r200x500": (200, 500, 4, 6)}.items():
        rng = np.random.default_rng(seed)
        trip = []
        for j in range(n):
            for r in rng.choice(m, size=per_col, replace=False):
                trip.append((int(r), j, float(rng.uniform(-1, 1))))
        off, col, val = csr(m, n, trip)
        A = np.zeros((m, n))
        for r in range(m):
            A[r, col[off[r]:off[r + 1]]] = val[off[r]:off[r + 1]]
        x0 = rng.uniform(0, 1, n) * (rng.uniform(0, 1, n) < 0.5)
        y0 = rng.uniform(-1, 1, m)
        s0 = rng.uniform(0, 1, n) * (x0 == 0)
        out[name] = (m, n, trip, list(A @ x0), list(A.T @ y0 + s0))
    return out


def main() -> None:
    L = O.load("ref")
    dp, i64p = C.POINTER(C.c_double), C.POINTER(C.c_int64)
    CP = C.POINTER(abi.PdlpCsr)
    L.ref_spectral_norm.argtypes = [CP, C.c_double, C.c_int32, dp]
    L.ref_kkt_error_standard.argtypes = [CP, dp, dp, dp, dp, dp]
    L.ref_p_s_norm_squared.argtypes = [CP, dp, dp, C.c_double, dp, dp, dp]
    L.ref_standard_pdhg.argtypes = [CP, dp, dp, C.c_double, C.c_double, C.c_double, C.c_int64, dp, dp, dp, i64p,
                                    C.c_int64, i64p, dp, dp, dp, dp, C.c_int64]
    P = abi.dptr
    out = {}
    for name, (m, n, trip, b, c) in fixtures().items():
        off, col, val = csr(m, n, trip)
        b, c = np.array(b, np.float64), np.array(c, np.float64)
        A = abi.PdlpCsr(num_rows=m, num_cols=n, nnz=len(val), row_offsets=abi.i64ptr(off),
                        col_indices=abi.i64ptr(col), values=P(val))
        norm = C.c_double(0.0)
        L.ref_spectral_norm(C.byref(A), 1e-12, 100000, C.byref(norm))
        s = 0.9 / (2.0 * norm.value)
        tol, limit = (1e-10, 400000) if m < 100 else (1e-8, 20000)
        cap = 1 << 14
        kkt, lens, cnt = np.zeros(cap), np.zeros(cap, np.int64), np.zeros(4, np.int64)
        xl, yl = np.zeros(n), np.zeros(m)
        ix, iy = np.zeros(REC * n), np.zeros(REC * m)
        rc = L.ref_standard_pdhg(C.byref(A), P(b), P(c), s, 0.5, tol, limit, None, None, P(kkt), abi.i64ptr(lens),
                                 cap, abi.i64ptr(cnt), P(xl), P(yl), P(ix), P(iy), REC)
        assert rc == 0
        ne = int(cnt[0])
        rng = np.random.default_rng(11)
        pts_x, pts_y = rng.uniform(-2, 2, (20, n)), rng.uniform(-2, 2, (20, m))
        kk, ps = np.zeros(20), np.zeros(20)
        for t in range(20):
            v = C.c_double(0.0)
            L.ref_kkt_error_standard(C.byref(A), P(b), P(c), P(pts_x[t]), P(pts_y[t]), C.byref(v))
            kk[t] = v.value
            L.ref_p_s_norm_squared(C.byref(A), P(b), P(c), s, P(pts_x[t]), P(pts_y[t]), C.byref(v))
            ps[t] = v.value
        rec = min(REC, int(cnt[1]))
        out.update({f"{name}/off": off, f"{name}/col": col, f"{name}/val": val, f"{name}/b": b, f"{name}/c": c,
                    f"{name}/norm": np.array([norm.value]), f"{name}/params": np.array([s, 0.5, tol, limit]),
                    f"{name}/kkt": kkt[:ne], f"{name}/lens": lens[:ne], f"{name}/counters": cnt,
                    f"{name}/x_last": xl, f"{name}/y_last": yl, f"{name}/iter_x": ix[:rec * n].reshape(rec, n),
                    f"{name}/iter_y": iy[:rec * m].reshape(rec, m), f"{name}/pts_x": pts_x, f"{name}/pts_y": pts_y,
                    f"{name}/kkt_pts": kk, f"{name}/ps_pts": ps})
        print(name, "norm", norm.value, "epochs", ne, "iterations", int(cnt[1]), "converged", int(cnt[2]))
    # the already-optimal chain (test_standard_form.cpp:112-127): z0 = (1, 1), tol disabled, 10 iterations
    off, col, val = csr(1, 1, [(0, 0, 1.0)])
    A = abi.PdlpCsr(num_rows=1, num_cols=1, nnz=1, row_offsets=abi.i64ptr(off), col_indices=abi.i64ptr(col),
                    values=P(val))
    one = np.ones(1)
    kkt, lens, cnt = np.zeros(64), np.zeros(64, np.int64), np.zeros(4, np.int64)
    xl, yl = np.zeros(1), np.zeros(1)
    assert L.ref_standard_pdhg(C.byref(A), P(one), P(one), 0.4, 0.5, -1.0, 10, P(one), P(one), P(kkt),
                               abi.i64ptr(lens), 64, abi.i64ptr(cnt), P(xl), P(yl), None, None, 0) == 0
    out.update({"chain/kkt": kkt[:cnt[0]], "chain/lens": lens[:cnt[0]], "chain/counters": cnt})
    # numerical failure: f4 with a step far beyond 1 / ||A|| (standard_form.hpp:177-180)
    off, col, val = csr(3, 5, fixtures()["f4"][2])
    b4, c4 = np.array(fixtures()["f4"][3]), np.array(fixtures()["f4"][4])
    A = abi.PdlpCsr(num_rows=3, num_cols=5, nnz=len(val), row_offsets=abi.i64ptr(off),
                    col_indices=abi.i64ptr(col), values=P(val))
    kkt, lens, cnt = np.zeros(64), np.zeros(64, np.int64), np.zeros(4, np.int64)
    xl, yl = np.zeros(5), np.zeros(3)
    assert L.ref_standard_pdhg(C.byref(A), P(b4), P(c4), 1e150, 0.5, 1e-12, 100000, None, None, P(kkt),
                               abi.i64ptr(lens), 64, abi.i64ptr(cnt), P(xl), P(yl), None, None, 0) == 0
    out.update({"fail/kkt": kkt[:cnt[0]], "fail/lens": lens[:cnt[0]], "fail/counters": cnt})
    np.savez_compressed(OUT, **out)
    print("wrote", OUT, "chain epochs", len(out["chain/kkt"]), "failure run", out["fail/counters"])


if __name__ == "__main__":
    main()
