# round-1 evidence: launch list (stream engine: ncu cannot see kernel nodes of
# conditional graphs), full captures of the hot kernels (cold + warm cache), bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01j
export PDLP_GRAPH=0
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01j/launches.csv python tools/profile_c2.py C2 > gpurun_out/r01j/launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"dual_kernel|primal_kernel" -s 200 -c 2 -o gpurun_out/r01j/prof_cold python tools/profile_c2.py C2 > gpurun_out/r01j/prof_cold.log 2>&1
timeout 900 ncu --set full --cache-control none --clock-control none --import-source on -k regex:"dual_kernel|primal_kernel|eval_" -s 200 -c 6 -o gpurun_out/r01j/prof_warm python tools/profile_c2.py C2 > gpurun_out/r01j/prof_warm.log 2>&1
unset PDLP_GRAPH
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r01j/bench.json 2> gpurun_out/r01j/bench.err
cat gpurun_out/r01j/bench.json
timeout 1500 python tools/bench_configs.py C1 C2 C3 C4 > gpurun_out/r01j/configs.jsonl 2> gpurun_out/r01j/configs.err
tail -8 gpurun_out/r01j/configs.err
ls -la gpurun_out/r01j
