# full regression + smoke + bench + configs (profiles refresh)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/final
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -4 | tee gpurun_out/final/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 | tee gpurun_out/final/smoke.txt
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err; cat gpurun_out/final/bench.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final/bench_ref.json 2>&1; cat gpurun_out/final/bench_ref.json
timeout 2400 python tools/bench_configs.py ${CONFIGS:-C1 C2 C3 C4} > gpurun_out/final/configs.jsonl 2> gpurun_out/final/configs.err; tail -6 gpurun_out/final/configs.err
