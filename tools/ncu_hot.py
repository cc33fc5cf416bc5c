"""Summarise an ncu source page (SASS): top instructions by warp-stall samples."""
import csv, sys, subprocess
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--launch-count", "1", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr) and r[2].isdigit()]
tot = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in data)
print("total samples", tot, "instructions", len(data))
for i, d in sorted(enumerate(data), key=lambda x: -int(x[1]["Warp Stall Sampling (All Samples)"] or 0))[:top]:
    s = int(d["Warp Stall Sampling (All Samples)"] or 0)
    print(f"{i:5d} {100*s/max(tot,1):5.1f}% {d['Source'].strip()[:90]}")
