cd $GRAFT_REPO_ROOT
export PDLP_GRAPH=0 PDLP_ITER_LIMIT=200
timeout 900 ncu --set full --cache-control none --clock-control none --import-source on -k regex:"dual_kernel|primal_kernel" -s 40 -c 2 -o gpurun_out/prof_c3 python tools/profile_c2.py C3 > gpurun_out/prof_c3.log 2>&1
tail -2 gpurun_out/prof_c3.log
