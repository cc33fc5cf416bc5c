cd $GRAFT_REPO_ROOT
for v in 0 1; do echo "=== DECIDE_SEP=$v"; PDLP_DECIDE_SEP=$v ENGINE=2 timeout 300 python tools/micro.py C2 2>&1 | grep -v copy; done
export PDLP_GRAPH=0
timeout 600 ncu --set full --cache-control none --clock-control none -k regex:"eval_" -s 8 -c 4 -o gpurun_out/prof_eval python tools/profile_c2.py C2 > gpurun_out/prof_eval.log 2>&1
tail -2 gpurun_out/prof_eval.log
