# C4 launch list with DRAM bytes of one timed dual group and one primal group (roofline.traffic)
cd $GRAFT_REPO_ROOT
D=gpurun_out/${TAG:-r02t}
mkdir -p $D
NCU_SOLVE=0 timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file $D/c4_launches.csv python tools/ncu_kernels.py C4 0 1 > $D/c4_launches.log 2>&1; tail -2 $D/c4_launches.log
