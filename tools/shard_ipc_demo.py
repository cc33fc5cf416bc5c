"""Row-sharded solve with one process per rank (the multi-GPU code path):
torch.distributed (gloo) carries only the CUDA-IPC blobs; the ranks then
exchange x' / y' slices and partials GPU-to-GPU inside the kernels, ordered by
the in-kernel epoch flags.

  python tools/shard_ipc_demo.py WORLD [--devices same|distinct] [--config NAME]

With --devices same (default, for a one-GPU box) every rank uses GPU 0 and the
driver time-slices the contexts; with distinct, rank r uses GPU r. Rank 0
checks the result against a single-rank solve planned with the same tile
breaks (bitwise) and prints "ipc ok".
"""
from __future__ import annotations

import argparse
import os
import socket
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def lp_for(name: str):
    from paper_2311_12180_b200 import generators

    if name == "small":
        return generators.random_lp(1500, 1500, 4000, 4, seed=11)
    return generators.config(name)


def main_rank(rank: int, world: int, port: int, distinct: bool, name: str, limit: int) -> None:
    import numpy as np
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2311_12180_b200 import SolverParams, solve, solve_distributed

    lp = lp_for(name)
    p = SolverParams(eps_optimal=1e-6, iteration_limit=limit, device=rank if distinct else 0)
    r = solve_distributed(lp, p)
    res = [None] * world
    dist.all_gather_object(res, (r.iterations, r.status.value, r.point.primal.tobytes(), r.point.dual.tobytes()))
    if rank == 0:
        ref = solve(lp, SolverParams(eps_optimal=1e-6, iteration_limit=limit, plan_world=world, device=0))
        ok = all(t == res[0] for t in res) and res[0][0] == ref.iterations and \
            res[0][2] == ref.point.primal.tobytes() and res[0][3] == ref.point.dual.tobytes()
        print(f"world {world}: {r.status} it {r.iterations} obj {r.info['primal_objective']:.12g} "
              f"ref it {ref.iterations} obj {ref.info['primal_objective']:.12g} "
              f"device_s {r.info['device_seconds']:.3f}", flush=True)
        print("ipc ok" if ok else "ipc MISMATCH", flush=True)
        if not ok:
            sys.exit(3)
    dist.barrier()
    dist.destroy_process_group()
    del np


def main() -> None:
    import torch.multiprocessing as mp

    ap = argparse.ArgumentParser()
    ap.add_argument("world", type=int)
    ap.add_argument("--devices", default="same", choices=["same", "distinct"])
    ap.add_argument("--config", default="small")
    ap.add_argument("--limit", type=int, default=640)
    a = ap.parse_args()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.spawn(main_rank, args=(a.world, port, a.devices == "distinct", a.config, a.limit), nprocs=a.world,
             join=True)


if __name__ == "__main__":
    main()
