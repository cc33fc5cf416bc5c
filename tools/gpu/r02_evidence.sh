# C4 evidence: per-launch DRAM traffic of the timed dual / primal groups, one full capture,
# occupancy variants of the panel sweep, C2 dual-kernel planner knobs, config parity prints
cd $GRAFT_REPO_ROOT
D=gpurun_out/${TAG:-r02o}
mkdir -p $D
NCU_SOLVE=0 timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file $D/c4_launches.csv python tools/ncu_kernels.py C4 0 1 > $D/c4_launches.log 2>&1; tail -2 $D/c4_launches.log
NCU_SOLVE=0 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"sweep_dual_final|sweep_pass" -s 2 -c 2 -o $D/c4_full python tools/ncu_kernels.py C4 0 > $D/c4_full.log 2>&1; tail -1 $D/c4_full.log
AB_ROUNDS=1 timeout 1500 python tools/ab_config.py C4 base "o5:x:" "o6:x:" "o5b:x:" > $D/ab_c4.jsonl 2> $D/ab_c4.err; cat $D/ab_c4.jsonl
AB_ITERS=2048 AB_ROUNDS=2 timeout 900 python tools/ab_config.py C2 base "lane8::PDLP_LANE_NNZ=8" "lane4::PDLP_LANE_NNZ=4" "w512::PDLP_WARP_MAX_ROW=512,PDLP_CHUNK_NNZ=512" > $D/ab_c2.jsonl 2> $D/ab_c2.err; cat $D/ab_c2.jsonl
timeout 2400 python -m pytest tests/test_gpu_configs.py -m gpu -q -s -k "iterates" > $D/configs_iterates.txt 2>&1; grep -E "worst|passed|failed" $D/configs_iterates.txt
