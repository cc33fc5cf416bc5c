"""Calibration microbenchmarks (dev tool): D2D copy bandwidth vs SpMV/iteration kernels on C2."""
import sys, os
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2311_12180_b200 import Solver, SolverParams, generators, abi

def copy_bw(nbytes):
    a = torch.empty(nbytes // 8, dtype=torch.float64, device="cuda"); b = torch.empty_like(a)
    for _ in range(3): b.copy_(a)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): b.copy_(a)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    return ms, 2 * nbytes / ms / 1e6
for mb in (36, 76, 128, 512):
    ms, gbs = copy_bw(mb << 20)
    print(f"copy {mb} MB (r+w {2*mb} MB): {ms*1e3:.1f} us {gbs:.0f} GB/s", flush=True)
lp = generators.config(sys.argv[1] if len(sys.argv) > 1 else "C2")
eng = int(os.environ.get("ENGINE", "2"))
s = Solver(lp, SolverParams(engine=eng))
r = s.solve()
r = s.solve()
print("solve", r.iterations, r.info["device_seconds"], "window", r.info["window_seconds"], "eval",
      r.info["eval_seconds"], "gap", r.info["device_seconds"] - r.info["window_seconds"] - r.info["eval_seconds"],
      flush=True)
for which, name in ((2, "spmv K"), (3, "spmv KT"), (0, "dual"), (1, "primal")):
    ms, by = s.time_kernel(which, 100)
    print(f"{name:8s} {ms*1e3:7.1f} us  {by/1e6:7.1f} MB  {by/ms/1e6:7.0f} GB/s", flush=True)
