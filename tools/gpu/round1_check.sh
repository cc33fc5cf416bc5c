set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 --no-cpu > gpurun_out/b_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:primal_kernel -s 50 -c 2 -o gpurun_out/prof_primal python bench.py --steps 1 --warmup 0 --no-cpu > gpurun_out/prof.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dual_kernel -s 50 -c 2 -o gpurun_out/prof_dual python bench.py --steps 1 --warmup 0 --no-cpu > gpurun_out/prof2.log 2>&1
ls -la gpurun_out
