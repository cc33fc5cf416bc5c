cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
for kn in "PDLP_NO_CONTIG=1 PDLP_NO_LAZY_KTY=1" "PDLP_NO_LAZY_KTY=1" "PDLP_NO_CONTIG=1" "X=1"; do
  echo "=== $kn"; env $kn ENGINE=2 timeout 300 python tools/micro.py C2 2>&1 | grep -v copy
done
echo "=== bench"; timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu 2>&1 | tail -1
