# A/B of library variants (tools/ab_config.py syntax) on a config, plus the panel/shard GPU tests
cd $GRAFT_REPO_ROOT
D=gpurun_out/${TAG:-r02p}
mkdir -p $D
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py -m gpu -q -x -s -k "${PYK:-panel or shard or coupling}" > $D/pytest.txt 2>&1; grep -E "passed|failed|values pushed" $D/pytest.txt
AB_ROUNDS=${ROUNDS:-1} timeout 2400 python tools/ab_config.py ${CFG:-C4} base "$@" > $D/ab.jsonl 2> $D/ab.err
cat $D/ab.jsonl; tail -3 $D/ab.err
