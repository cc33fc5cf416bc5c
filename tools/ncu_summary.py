"""Summarise the ncu evidence of one GPU call into profiles/ (committed).

  python tools/ncu_summary.py r01 gpurun_out

Reads (all optional):
  <dir>/launches.csv          `ncu --metrics gpu__time_duration.sum` launch list
  <dir>/prof_<name>.ncu-rep   `ncu --set full` captures of the hot kernels
and writes
  profiles/<tag>_launches.md  per-kernel count / total / share of the launch list
  profiles/<tag>_ncu.json     per-capture DRAM bytes, time, occupancy, stalls
  profiles/ncu_summary.json   latest per-kernel DRAM bytes per launch (bench.py
                              reads it for roofline.traffic)
"""
from __future__ import annotations

import collections
import csv
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
KEYS = {
    "gpu__time_duration.sum": "time",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_peak",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__occupancy_limit_registers": "ctas_per_sm_reg_limit",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio": "stall_long_scoreboard",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio": "stall_barrier",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio": "stall_short_scoreboard",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio": "stall_wait",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0,
         "msecond": 1e3}


def launches(path: Path) -> list[dict]:
    rows = list(csv.reader(path.read_text().splitlines()))
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[start]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot, cnt = collections.Counter(), collections.Counter()
    for r in rows[start + 1:]:
        if len(r) < len(hdr):
            continue
        us = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
        name = r[ki].split("(")[0].replace("void ", "")
        tot[name] += us
        cnt[name] += 1
    s = sum(tot.values())
    return [{"kernel": k, "launches": cnt[k], "total_us": v, "share": v / s, "avg_us": v / cnt[k]}
            for k, v in tot.most_common()]


def capture(rep: Path) -> list[dict]:
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")}
        for k, short in KEYS.items():
            if k in hdr:
                i = hdr.index(k)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                if short.startswith("dram_r") or short.startswith("dram_w"):
                    v *= SCALE.get(units[i], 1.0)
                elif short == "time":
                    v *= SCALE.get(units[i], 1.0)
                d[short] = v
        if "dram_read" in d:
            d["dram_bytes_per_launch"] = d["dram_read"] + d.get("dram_write", 0.0)
        res.append(d)
    return res


def main() -> None:
    tag, src = sys.argv[1], Path(sys.argv[2])
    prof = ROOT / "profiles"
    prof.mkdir(exist_ok=True)
    if (src / "launches.csv").exists():
        ls = launches(src / "launches.csv")
        lines = [f"# {tag}: ncu launch list (cold-cache, serialised: compare shares, not absolutes)", "",
                 "| kernel | launches | total µs | share | avg µs |", "|---|---|---|---|---|"]
        lines += [f"| `{d['kernel']}` | {d['launches']} | {d['total_us']:.1f} | {100 * d['share']:.1f}% | "
                  f"{d['avg_us']:.2f} |" for d in ls[:25]]
        (prof / f"{tag}_launches.md").write_text("\n".join(lines) + "\n")
    caps = {}
    for rep in sorted(src.glob("prof_*.ncu-rep")):
        caps[rep.stem[5:]] = capture(rep)
    if caps:
        (prof / f"{tag}_ncu.json").write_text(json.dumps(caps, indent=1))
        summary_path = prof / "ncu_summary.json"
        summary = json.loads(summary_path.read_text()) if summary_path.exists() else {}
        # the cold-cache capture (caches flushed before each kernel) wins when
        # present: roofline.traffic is the conservative DRAM figure
        for name, lst in sorted(caps.items(), key=lambda kv: kv[0] == "cold"):
            by_kernel: dict = {}
            for d in lst:
                if "dram_bytes_per_launch" in d:
                    base = d["kernel"].split("<")[0].split("::")[-1]
                    by_kernel.setdefault(base, []).append(d)
            for base, ds in by_kernel.items():
                summary[base] = {
                    "dram_bytes_per_launch": sum(d["dram_bytes_per_launch"] for d in ds) / len(ds),
                    "time_us": sum(d.get("time", 0.0) for d in ds) / len(ds), "launches": len(ds),
                    "capture": name, "round": tag, "source": f"profiles/{tag}_ncu.json"}
        summary_path.write_text(json.dumps(summary, indent=1, sort_keys=True))
    print("wrote", sorted(p.name for p in prof.glob(f"{tag}_*")))


if __name__ == "__main__":
    main()
