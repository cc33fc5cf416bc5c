"""Summarise an ncu report (dev tool): per launch, time, DRAM bytes and
throughput, L2 hit rate and throughput, warp occupancy and the top stall
reasons.

  python tools/ncu_summary_rep.py gpurun_out/x.ncu-rep
"""
import csv
import io
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
           "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size", "launch__registers_per_thread",
           "lts__t_sectors_srcunit_tex_op_read.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum"]

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
stall = [i for i, h in enumerate(hdr) if h.startswith("smsp__average_warp_latency_issue_stalled_") or
         h.startswith("smsp__pcsamp_warps_issue_stalled_")]
for r in rows[2:]:
    print(r[hdr.index("Kernel Name")][:70])
    for m in METRICS:
        if m in hdr:
            print(f"  {m} = {r[hdr.index(m)]} {rows[1][hdr.index(m)]}")
    st = []
    for i in stall:
        try:
            st.append((float(r[i]), hdr[i]))
        except ValueError:
            pass
    tot = sum(v for v, h in st if "pcsamp" in h and not h.endswith("_not_issued"))
    for v, h in sorted(st, reverse=True)[:8]:
        print(f"  {h} = {v:g}" + (f" ({100 * v / tot:.0f}%)" if tot and "pcsamp" in h else ""))
