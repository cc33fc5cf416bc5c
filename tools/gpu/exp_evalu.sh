cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for c in C1 C2 C3; do echo "=== $c"; ENGINE=2 timeout 300 python tools/micro.py $c 2>&1 | grep solve; done
