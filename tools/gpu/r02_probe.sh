# panel geometry probe: event times, then the same under ncu (DRAM bytes per sweep launch)
cd $GRAFT_REPO_ROOT
D=gpurun_out/${TAG:-r02h}
mkdir -p $D
timeout 1200 python tools/panel_probe.py ${CFG:-C4} "$@" > $D/probe.jsonl 2> $D/probe.err; cat $D/probe.jsonl; tail -3 $D/probe.err
PROBE_REPS=1 timeout 2400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none -k regex:"sweep_kernel" --csv --log-file $D/probe_ncu.csv python tools/panel_probe.py ${CFG:-C4} "$@" > $D/probe_ncu.log 2>&1
python - $D/probe_ncu.csv <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
ii = h.index("ID")
cur = {}
for r in rows[1:]:
    cur.setdefault(r[ii], {"k": r[ki][:40]})[r[mi]] = r[vi]
for i, d in cur.items():
    print(i, d.get("gpu__time_duration.sum"), "read", d.get("dram__bytes_read.sum"), "write", d.get("dram__bytes_write.sum"), "hit", d.get("lts__t_sector_hit_rate.pct"), "l2rd", d.get("lts__t_sectors_srcunit_tex_op_read.sum"))
PY
