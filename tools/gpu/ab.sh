cd $GRAFT_REPO_ROOT
for c in ${CFGS:-C2 C3}; do timeout 1200 python tools/ab_kernels.py $c ${VARIANTS}; done
