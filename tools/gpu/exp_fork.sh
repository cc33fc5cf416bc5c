cd $GRAFT_REPO_ROOT
for kn in "PDLP_NO_EVAL_FORK=1" "X=1"; do for c in C2 C3; do echo "=== $c $kn"; env $kn ENGINE=2 timeout 300 python tools/micro.py $c 2>&1 | grep solve; done; done
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
