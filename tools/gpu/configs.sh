# per-config measurements (tools/bench_configs.py) -> gpurun_out/configs.jsonl
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv
timeout 1500 python tools/bench_configs.py ${CONFIGS:-C1 C2 C3 C4} > gpurun_out/configs.jsonl 2> gpurun_out/configs.err
tail -20 gpurun_out/configs.err
cat gpurun_out/configs.jsonl
