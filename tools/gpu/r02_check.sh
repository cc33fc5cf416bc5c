# round-2 state check: GPU tests, smoke, bench (C4 headline), reference arm
cd $GRAFT_REPO_ROOT
D=gpurun_out/${TAG:-r02a}
mkdir -p $D
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $D/gpu.txt
timeout 3000 python -m pytest tests -m gpu -q ${PYTEST_K:+-k "$PYTEST_K"} > $D/pytest_gpu.txt 2>&1; tail -15 $D/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.txt 2>&1; tail -2 $D/smoke.txt
timeout 1500 python bench.py --steps ${STEPS:-5} --warmup 3 > $D/bench.json 2> $D/bench.err; cat $D/bench.json; tail -5 $D/bench.err
if [ -z "$NOREF" ]; then timeout 1500 python bench.py --impl reference --steps 2 --warmup 1 > $D/bench_ref.json 2> $D/bench_ref.err; cat $D/bench_ref.json; tail -3 $D/bench_ref.err; fi
