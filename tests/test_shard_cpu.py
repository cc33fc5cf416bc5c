"""CPU tests (no GPU) of the row-sharding host logic: the
partition every rank computes (libpdlp_b200.so pdlp_plan_shards, host-only),
its agreement across ranks of a real world_size-2 torch.distributed group over
gloo, the blob exchange protocol solve_distributed uses, the library's gather
masks (pdlp_plan_exchange, the host twin of the device masks), and the algebra
of one sharded PDHG trial in which each rank sends every x' value only to the
ranks its mask names (the coupling-only exchange): the ranks' slices reproduce
the unsharded trial exactly."""
from __future__ import annotations

import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2311_12180_b200 import SolverParams, abi, generators, plan_exchange, plan_shards
from paper_2311_12180_b200.api import load_library
from tests.helpers import stacked_k


def lps():
    return {"C1": generators.config("C1"), "transport": generators.transport_lp(60, 90, seed=3),
            "multicommodity": generators.multicommodity_lp(300, 1500, 4, seed=2),
            "staircase": generators.staircase_lp(4, 600, 150, 150, seed=4)}


@pytest.mark.parametrize("world", [2, 3, 4, 8])
@pytest.mark.parametrize("name", ["C1", "transport", "multicommodity", "staircase"])
def test_plan_shards_partition(name, world):
    lp = lps()[name]
    kc, ktc = plan_shards(lp, world)
    K = stacked_k(lp)
    for cuts, rows, rp in ((kc, K.num_rows, K.row_offsets),
                           (ktc, lp.num_variables, np.concatenate([[0], np.cumsum(np.bincount(
                               K.col_indices, minlength=lp.num_variables))]))):
        assert cuts[0] == 0 and cuts[-1] == rows
        assert (np.diff(cuts) > 0).all()
        assert all(c % 4 == 0 for c in cuts[1:-1])  # 4-row aligned tile starts
        w = rp[cuts[1:]] + cuts[1:] - rp[cuts[:-1]] - cuts[:-1]  # nnz + rows per shard
        assert w.max() <= (rp[-1] + rows) / world * 1.25 + rp[1:].max() - rp[:-1].min() + 8


def test_plan_shards_rejects_too_many_ranks():
    lp = generators.small_random_lp(5, 2, 2, seed=1)
    with pytest.raises(ValueError, match="cannot be split"):
        plan_shards(lp, 8)


def test_invalid_shard_params_are_einval_without_gpu():
    lib = load_library()
    lp = generators.small_random_lp(6, 3, 2, seed=1)
    for kw in (dict(world_size=2, rank=2), dict(world_size=9), dict(world_size=2, mode=1),
               dict(world_size=2, engine=abi.ENGINE_PERSISTENT), dict(engine=abi.ENGINE_PERSISTENT)):
        h = C.c_void_p()
        lpa, pa = lp.to_abi(), SolverParams(**kw).to_abi()
        assert lib.pdlp_create(C.byref(lpa), C.byref(pa), C.byref(h)) == abi.PDLP_EINVAL, kw


def rows_dot(K, r0: int, r1: int, x: np.ndarray) -> np.ndarray:
    """(K x)[r0:r1] summed sequentially per row, as spmv (sparse_matrix.hpp:
    123-131): the same rounding on every rank and in the unsharded check."""
    out = np.zeros(r1 - r0)
    for r in range(r0, r1):
        acc = 0.0
        for k in range(int(K.row_offsets[r]), int(K.row_offsets[r + 1])):
            acc += float(K.values[k]) * float(x[int(K.col_indices[k])])
        out[r - r0] = acc
    return out


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank: int, world: int, port: int, out, name: str = "C1"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lp = lps()[name]  # every rank generates the same seeded instance
        kc, ktc = plan_shards(lp, world)
        ex = plan_exchange(lp, world)  # the library's gather masks (host twin of the device's)
        cuts = [None] * world
        dist.all_gather_object(cuts, (kc.tolist(), ktc.tolist(), ex["pushed"].tolist()))
        # the blob exchange of solve_distributed: fixed-size byte strings in rank order
        size = int(load_library().pdlp_shard_blob_size())
        blob = bytes([rank]) * size
        blobs = [None] * world
        dist.all_gather_object(blobs, blob)

        # one sharded PDHG trial (solver.hpp:404-415) on the unscaled instance:
        # rank p owns rows [kc[p], kc[p+1]) of K and columns [ktc[p], ktc[p+1]),
        # and sends each x' / y' value only to the ranks its mask names; values
        # nobody sent stay NaN, so a missing one would poison the result
        K = stacked_k(lp)
        Kd = K.to_dense()
        rng = np.random.default_rng(7)
        x, y = rng.uniform(0, 1, lp.num_variables), rng.uniform(-1, 1, lp.num_constraints)
        q = np.concatenate([lp.inequality_rhs, lp.equality_rhs])
        tau = sigma = 0.3
        kty = Kd.T @ y
        c0, c1 = ktc[rank], ktc[rank + 1]
        x_own = np.clip(x[c0:c1] - tau * (lp.objective[c0:c1] - kty[c0:c1]), lp.lower[c0:c1], lp.upper[c0:c1])
        sends = [{int(j): float(x_own[j - c0]) for j in range(c0, c1) if (ex["xmask"][j] >> dst) & 1}
                 for dst in range(world)]
        got = [None] * world
        dist.all_gather_object(got, sends)
        x_new = np.full(lp.num_variables, np.nan)
        x_new[c0:c1] = x_own
        for src in range(world):
            for j, v in got[src][rank].items():
                x_new[j] = v
        r0, r1 = kc[rank], kc[rank + 1]
        kx = rows_dot(K, r0, r1, x)
        kxn_own = rows_dot(K, r0, r1, x_new)  # a NaN here would mean a value never arrived
        needed = np.unique(K.col_indices[K.row_offsets[r0]:K.row_offsets[r1]])
        assert not np.isnan(x_new[needed]).any()  # every column a local row touches arrived
        y_own = y[r0:r1] + sigma * (q[r0:r1] - 2.0 * kxn_own + kx)
        y_own[: max(0, min(r1, lp.num_inequalities) - r0)] = np.maximum(
            y_own[: max(0, min(r1, lp.num_inequalities) - r0)], 0.0)
        dy2 = float(((y_own - y[r0:r1]) ** 2).sum())
        ys = [None] * world
        dist.all_gather_object(ys, (y_own, dy2))
        sent = sum(len(d) for d in sends) - len(sends[rank])
        others = ((1 << world) - 1) & ~(1 << rank)
        x_part = sum(bin(int(ex["xmask"][j]) & others).count("1") for j in range(c0, c1))
        y_part = sum(bin(int(ex["ymask"][i]) & others).count("1") for i in range(r0, r1))
        out.put((rank, cuts, [b[0] for b in blobs], len(blobs[0]), np.concatenate([v[0] for v in ys]),
                 [v[1] for v in ys], x_new[needed], needed, (sent, x_part, y_part)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["C1", "staircase"])
def test_gloo_world2_partition_and_sharded_trial(name):
    world = 2
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, out, name)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([out.get(timeout=240) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # every rank computed the same partition and exchange plan, and saw every blob in rank order
    assert res[0][1] == res[1][1]
    assert res[0][2] == [0, 1] and res[1][2] == [0, 1]
    assert res[0][3] == int(load_library().pdlp_shard_blob_size())
    # each rank sent exactly the x' values its masks name, and the library's
    # per-rank count is those plus the y' values its masks name
    pushed = res[0][1][0][2]
    for r in res:
        sent, x_part, y_part = r[8]
        assert sent == x_part and x_part + y_part == pushed[r[0]]
    # the gathered trial equals the unsharded trial
    lp = lps()[name]
    Ks = stacked_k(lp)
    K = Ks.to_dense()
    rng = np.random.default_rng(7)
    x, y = rng.uniform(0, 1, lp.num_variables), rng.uniform(-1, 1, lp.num_constraints)
    q = np.concatenate([lp.inequality_rhs, lp.equality_rhs])
    xn = np.clip(x - 0.3 * (lp.objective - K.T @ y), lp.lower, lp.upper)
    m = lp.num_constraints
    yn = y + 0.3 * (q - 2.0 * rows_dot(Ks, 0, m, xn) + rows_dot(Ks, 0, m, x))
    yn[: lp.num_inequalities] = np.maximum(yn[: lp.num_inequalities], 0.0)
    for r in res:
        assert np.array_equal(r[6], xn[r[7]])
        assert np.array_equal(r[4], yn)
    assert np.isclose(sum(res[0][5]), ((yn - y) ** 2).sum(), rtol=1e-12)
