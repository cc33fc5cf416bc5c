# dev sweep: engines and planner knobs on C2 / C1 (numbers are exploratory, not bench values)
cd $GRAFT_REPO_ROOT
for eng in 2 1; do echo "=== C2 ENGINE=$eng"; ENGINE=$eng timeout 300 python tools/micro.py C2 2>&1 | grep -v copy; done
for ln in 4 8 32; do echo "=== C2 LANE_NNZ=$ln"; PDLP_LANE_NNZ=$ln ENGINE=2 timeout 300 python tools/micro.py C2 2>&1 | grep -v copy; done
echo "=== C1"; ENGINE=2 timeout 300 python tools/micro.py C1 2>&1
echo "=== C1 persistent"; ENGINE=1 timeout 300 python tools/micro.py C1 2>&1 | grep -v copy
