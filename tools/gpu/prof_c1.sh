cd $GRAFT_REPO_ROOT
export PDLP_GRAPH=0 PDLP_ITER_LIMIT=300
timeout 900 ncu --set full --cache-control none --clock-control none --import-source on -k regex:"dual_kernel|primal_kernel" -s 100 -c 4 -o gpurun_out/prof_c1 python tools/profile_c2.py C1 > gpurun_out/prof_c1.log 2>&1
tail -2 gpurun_out/prof_c1.log
ENGINE=2 timeout 300 python tools/micro.py C1 2>&1 | grep -v copy
PDLP_NO_PDL=1 ENGINE=2 timeout 300 python tools/micro.py C1 2>&1 | grep -v copy
