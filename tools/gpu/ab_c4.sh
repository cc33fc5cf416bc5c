cd $GRAFT_REPO_ROOT
AB_ROUNDS=2 timeout 1500 python tools/ab_config.py C4 "base" "c1k6:x" "c1k5:x" "c2k3:x" "c2k5:x" "kt48::PDLP_PANEL_MB_T=48" "k64::PDLP_PANEL_MB_K=64" > gpurun_out/ab_c4.jsonl 2> gpurun_out/ab_c4.err
cat gpurun_out/ab_c4.jsonl
