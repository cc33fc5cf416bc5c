cd $GRAFT_REPO_ROOT
free -g | head -2; nvidia-smi --query-gpu=memory.total,memory.used --format=csv
timeout 2400 python tools/bench_configs.py C5 > gpurun_out/c5.jsonl 2> gpurun_out/c5.err
tail -5 gpurun_out/c5.err; cat gpurun_out/c5.jsonl | cut -c1-2000
