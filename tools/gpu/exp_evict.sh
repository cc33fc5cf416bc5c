cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
for c in C2 C3; do echo "=== $c"; ENGINE=2 timeout 300 python tools/micro.py $c 2>&1 | grep -v copy; done
timeout 900 python tools/bench_configs.py C4 2>&1 | tail -1 | cut -c1-1500
