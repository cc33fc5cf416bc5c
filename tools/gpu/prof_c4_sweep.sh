# ncu of the C4 panel sweeps (stream engine so ncu sees every launch)
cd $GRAFT_REPO_ROOT
export PDLP_ITER_LIMIT=64
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"sweep_pass" -s 40 -c 3 -o gpurun_out/prof_c4s2 python tools/profile_c2.py C4 > gpurun_out/prof_c4s2.log 2>&1
tail -2 gpurun_out/prof_c4s2.log
