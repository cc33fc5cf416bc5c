cd $GRAFT_REPO_ROOT
for c in C1 C2; do echo "=== $c"; ENGINE=2 timeout 300 python tools/micro.py $c 2>&1 | grep -v copy; done
