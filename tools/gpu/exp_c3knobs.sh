cd $GRAFT_REPO_ROOT
for kn in "X=1" "PDLP_STREAM_MAX_ROW=64" "PDLP_STREAM_MAX_ROW=128" "PDLP_STREAM_MAX_ROW=256"; do echo "=== C3 $kn"; env $kn ENGINE=2 timeout 300 python tools/micro.py C3 2>&1 | grep -v copy; done
