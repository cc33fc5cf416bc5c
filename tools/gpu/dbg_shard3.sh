cd $GRAFT_REPO_ROOT
for kn in "PDLP_STREAM_MAX_ROW=32" "PDLP_STREAM_MAX_ROW=64" "X=1"; do
echo "== $kn"; env $kn timeout 300 python -m pytest tests/test_gpu_shard.py -q -x -k "skewed" 2>&1 | tail -1
done
PDLP_DECIDE_SEP=1 timeout 300 python -m pytest tests/test_gpu_shard.py -q -x -k "skewed" 2>&1 | tail -1
