# last pass of the round: C4 launch list (roofline.traffic), GPU tests, smoke, bench, reference arm
cd $GRAFT_REPO_ROOT
D=gpurun_out/r02last
mkdir -p $D
NCU_SOLVE=0 timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file $D/c4_launches.csv python tools/ncu_kernels.py C4 0 1 > $D/c4_launches.log 2>&1
TAG=r02last bash tools/gpu/r02_full.sh
