"""Per-trial exchange volume of a row-sharded solve (dev tool; needs a GPU,
one rank's handle at a time): for each config and world size, every rank's
x' / y' values pushed to peers with the gather masks, against an all-to-all
push (pdlp_shard_exchange). No linking and no solve: the masks are built at
create time.

  python tools/shard_volume.py C4 C5 > gpurun_out/shard_volume.jsonl
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2311_12180_b200 import Solver, SolverParams, generators  # noqa: E402

for cfg in sys.argv[1:]:
    lp = generators.config(cfg)
    for world in (2, 4, 8):
        pushed = a2a = 0
        per = []
        for rank in range(world):
            with Solver(lp, SolverParams(world_size=world, rank=rank)) as s:
                e = s.shard_exchange()
                pushed += e["pushed"]
                a2a += e["all_to_all"]
                per.append(e["pushed"])
        print(json.dumps({"config": cfg, "world": world, "pushed_values_per_trial": pushed,
                          "all_to_all_values_per_trial": a2a, "fraction": pushed / a2a,
                          "pushed_bytes_per_trial_per_rank_max": 8 * max(per)}), flush=True)
    del lp
