# warm-cache ncu capture of C2's dual_kernel (stream engine), source-level
cd $GRAFT_REPO_ROOT
export PDLP_GRAPH=0 PDLP_ITER_LIMIT=300
timeout 900 ncu --set full --cache-control none --clock-control none --import-source on -k regex:"dual_kernel" -s 100 -c 2 -o gpurun_out/prof_dual python tools/profile_c2.py C2 > gpurun_out/prof_dual.log 2>&1
tail -3 gpurun_out/prof_dual.log
