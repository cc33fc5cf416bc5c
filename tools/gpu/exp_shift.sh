cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for kn in "PDLP_NO_ROW_GROUPS=1" "X=1" "PDLP_CONTIG=1"; do echo "=== C2 $kn"; env $kn ENGINE=2 timeout 300 python tools/micro.py C2 2>&1 | grep -v copy; done
