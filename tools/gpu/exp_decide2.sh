cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for v in 0 1 2; do echo "=== DECIDE_SEP=$v"; PDLP_DECIDE_SEP=$v ENGINE=2 timeout 300 python tools/micro.py C2 2>&1 | grep -v copy; done
for v in 0 2; do echo "=== C1 DECIDE_SEP=$v"; PDLP_DECIDE_SEP=$v ENGINE=2 timeout 300 python tools/micro.py C1 2>&1 | grep -v copy; done
