# warm-cache ncu captures of the C2 iteration kernels (stream engine so ncu sees them)
cd $GRAFT_REPO_ROOT
export PDLP_GRAPH=0
timeout 600 ncu --set full --cache-control none --clock-control none --import-source on -k regex:"dual_kernel|primal_kernel|spmv_kernel" -s 60 -c 6 -o gpurun_out/prof_warm python tools/profile_c2.py C2 > gpurun_out/prof_warm.log 2>&1
tail -3 gpurun_out/prof_warm.log
# knob sweep on the dual side: rows of 1000 as WARP (lane groups) vs CHUNK tiles
for kn in "PDLP_WARP_MAX_ROW=512" "PDLP_WARP_MAX_ROW=512 PDLP_CHUNK_NNZ=512" "PDLP_LANE_NNZ=16"; do
  echo "=== $kn"; env $kn ENGINE=2 timeout 300 python tools/micro.py C2 2>&1 | grep -v copy
done
