# full GPU regression: all gpu tests, then the bench line
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -25
echo "=== bench"
timeout 600 python bench.py --steps 5 --warmup 3 2>&1 | tail -3
