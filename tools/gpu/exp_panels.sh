cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "panels" 2>&1 | tail -3
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
PDLP_TRACE_SETUP=1 timeout 1200 python tools/bench_configs.py C4 > gpurun_out/c4p.jsonl 2> gpurun_out/c4p.err; grep -E "panels|C4" gpurun_out/c4p.err | head; cut -c1-1600 gpurun_out/c4p.jsonl
