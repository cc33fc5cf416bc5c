# GPU check of the sharded path + regression suite
cd $GRAFT_REPO_ROOT
PDLP_IPC_TEST=0 timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -30
echo "=== IPC demo"
timeout 300 python tools/shard_ipc_demo.py 2 --limit 320 2>&1 | tail -20
echo "=== bench"
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu 2>&1 | tail -3
