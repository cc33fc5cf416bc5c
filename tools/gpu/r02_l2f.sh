cd $GRAFT_REPO_ROOT
D=gpurun_out/${TAG:-r02z}
mkdir -p $D
AB_ROUNDS=1 timeout 2400 python tools/ab_config.py C4 base "f32::PDLP_L2_FETCH=32" "f64::PDLP_L2_FETCH=64" "f128::PDLP_L2_FETCH=128" "nopanf32::PDLP_PANELS=0,PDLP_L2_FETCH=32" > $D/ab_c4.jsonl 2> $D/ab_c4.err; cat $D/ab_c4.jsonl
AB_ITERS=2048 AB_ROUNDS=1 timeout 900 python tools/ab_config.py C2 base "f32::PDLP_L2_FETCH=32" "f64::PDLP_L2_FETCH=64" > $D/ab_c2.jsonl 2> $D/ab_c2.err; cat $D/ab_c2.jsonl
