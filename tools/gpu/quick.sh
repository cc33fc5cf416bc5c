# quick regression + C2 numbers + configs C3/C4 (decide kernel)
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
echo "=== micro C2"; ENGINE=2 timeout 300 python tools/micro.py C2 2>&1 | grep -v copy
echo "=== bench"; timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu 2>&1 | tail -1
echo "=== configs"; timeout 1500 python tools/bench_configs.py ${CONFIGS:-C1 C3 C4} > gpurun_out/configs2.jsonl 2> gpurun_out/configs2.err; tail -4 gpurun_out/configs2.err
