# round-2 regression: GPU tests, smoke, bench (N=1), a 2-rank sharded bench on one GPU (C1, time-sliced), reference arm
cd $GRAFT_REPO_ROOT
D=gpurun_out/${TAG:-r02n}
mkdir -p $D
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $D/gpu.txt
timeout 3000 python -m pytest tests -m gpu -q ${PYK:+-k "$PYK"} > $D/pytest_gpu.txt 2>&1; tail -6 $D/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.txt 2>&1; tail -2 $D/smoke.txt
timeout 1500 python bench.py --steps ${STEPS:-5} --warmup 3 > $D/bench.json 2> $D/bench.err; cat $D/bench.json; tail -3 $D/bench.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 1 --config C1 --no-cpu > $D/bench_shard2_c1.json 2> $D/bench_shard2_c1.err; cat $D/bench_shard2_c1.json; tail -3 $D/bench_shard2_c1.err
if [ -z "$NOREF" ]; then timeout 1500 python bench.py --impl reference --steps 2 --warmup 1 > $D/bench_ref.json 2> $D/bench_ref.err; cat $D/bench_ref.json; tail -3 $D/bench_ref.err; fi
