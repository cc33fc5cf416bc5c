cd $GRAFT_REPO_ROOT
export PDLP_GRAPH=0 PDLP_ITER_LIMIT=64
timeout 1200 ncu --set full --clock-control none -k regex:"panel_spmv|combine" -s 20 -c 4 -o gpurun_out/prof_c4p python tools/profile_c2.py C4 > gpurun_out/prof_c4p.log 2>&1
tail -2 gpurun_out/prof_c4p.log
