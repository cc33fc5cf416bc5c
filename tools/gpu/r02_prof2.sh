# C4: ncu --set full of one dual SpMV pass, the dual final and the primal final (accept); shard volumes; occupancy variants
cd $GRAFT_REPO_ROOT
D=gpurun_out/${TAG:-r02r}
mkdir -p $D
NCU_SOLVE=0 timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"sweep_pass_kernel|sweep_dual_final|sweep_primal_final" -s 14 -c 10 -o $D/c4_full python tools/ncu_kernels.py C4 0 1 > $D/c4_full.log 2>&1; tail -1 $D/c4_full.log
timeout 1500 python tools/shard_volume.py C4 C5 > $D/shard_volume.jsonl 2> $D/shard_volume.err; cat $D/shard_volume.jsonl; tail -2 $D/shard_volume.err
AB_ROUNDS=1 timeout 1500 python tools/ab_config.py C4 base "p8:x:" "p7:x:" > $D/ab.jsonl 2> $D/ab.err; cat $D/ab.jsonl
