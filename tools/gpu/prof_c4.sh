cd $GRAFT_REPO_ROOT
export PDLP_GRAPH=0 PDLP_ITER_LIMIT=64
timeout 1200 ncu --set full --clock-control none -k regex:"dual_kernel|primal_kernel" -s 40 -c 2 -o gpurun_out/prof_c4 python tools/profile_c2.py C4 > gpurun_out/prof_c4.log 2>&1
tail -3 gpurun_out/prof_c4.log
