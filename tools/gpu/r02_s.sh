cd $GRAFT_REPO_ROOT
D=gpurun_out/${TAG:-r02s}
mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -s -k "small_tile_band or column_panel" > $D/pytest.txt 2>&1; grep -E "passed|failed|nnz|Error" $D/pytest.txt | head
timeout 900 python tools/setup_trace.py C4 > $D/setup_trace.txt 2>&1; cat $D/setup_trace.txt | tail -40
timeout 1500 python bench.py --steps 5 --warmup 3 > $D/bench.json 2> $D/bench.err; cat $D/bench.json; tail -3 $D/bench.err
