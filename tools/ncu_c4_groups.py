"""Summarise an ncu launch list of `tools/ncu_kernels.py C4 0 1` (dev tool):
the last timed dual group (panel passes + dual final) and primal group
(panel passes + primal final), per launch and in total, into
profiles/<tag>_c4_launches.md, and the group totals into
profiles/ncu_summary.json["C4"] (bench.py's roofline.traffic).

  python tools/ncu_c4_groups.py gpurun_out/r02t/c4_launches.csv r02t
"""
import csv
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3}

path, tag = sys.argv[1], sys.argv[2]
rows = [r for r in csv.reader(open(path)) if len(r) > 10]
h = rows[0]
ki, mi, vi, ii, ui = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID", "Metric Unit"))
L = {}
for r in rows[1:]:
    d = L.setdefault(int(r[ii]), {"k": r[ki]})
    d[r[mi]] = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1)
ids = sorted(L)
dual = [i for i in ids if "sweep_pass_kernel<0>" in L[i]["k"] or "sweep_dual_final" in L[i]["k"]][-7:]
prim = [i for i in ids if "sweep_pass_kernel<1>" in L[i]["k"] or "sweep_primal_final" in L[i]["k"]][-3:]
out = [f"# C4 iteration kernels, ncu launch list ({tag})", "",
       "`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,"
       "dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none` over `NCU_SOLVE=0 python "
       "tools/ncu_kernels.py C4 0 1` (one timed dual group, then one timed primal group in accept mode). "
       "Serialised and cold per launch: compare shares and bytes, not absolute times.", "",
       "| launch | kernel | µs | DRAM MB | L2 hit % | DRAM % of peak |", "|---|---|---|---|---|---|"]
tot = {}
for name, g in (("dual", dual), ("primal", prim)):
    t = b = 0.0
    for i in g:
        d = L[i]
        us = d["gpu__time_duration.sum"] / 1e3
        mb = (d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]) / 1e6
        t += us
        b += mb
        out.append(f"| {i} | {d['k'].split('(')[0]} | {us:.1f} | {mb:.1f} | {d['lts__t_sector_hit_rate.pct']:.1f} | "
                   f"{d['dram__throughput.avg.pct_of_peak_sustained_elapsed']:.1f} |")
    out.append(f"| **{name} group** | {len(g)} launches | **{t:.1f}** | **{b:.1f}** | | |")
    tot[name] = {"dram_bytes_per_launch": b * 1e6, "time_us": t, "launches": len(g)}
(ROOT / "profiles" / f"{tag}_c4_launches.md").write_text("\n".join(out) + "\n")
sp = ROOT / "profiles" / "ncu_summary.json"
s = json.loads(sp.read_text())
s["C4"] = {k: {**v, "capture": "cold, serialised", "round": tag, "source": f"profiles/{tag}_c4_launches.md"}
           for k, v in tot.items()}
sp.write_text(json.dumps(s, indent=1, sort_keys=True) + "\n")
print(json.dumps(tot))
