set -x
free -g; nproc; lscpu | head -20
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
./tools/micro/l2_gather > gpurun_out/l2_gather.txt 2>&1
PDLP_TRACE_SETUP=1 timeout 900 python tools/bench_configs.py C4 > gpurun_out/c4_base.jsonl 2> gpurun_out/c4_base.err
tail -5 gpurun_out/c4_base.err
