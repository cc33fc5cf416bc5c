# banded panels: parity of the sweep, then a C4 A/B over variants given as arguments
# (tools/ab_config.py syntax: name[:defines[:ENV=V,...]]); TAG names the output dir
cd $GRAFT_REPO_ROOT
D=gpurun_out/${TAG:-r02c}
mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "${PYK:-panel}" > $D/pytest_panels.txt 2>&1; tail -5 $D/pytest_panels.txt
AB_ROUNDS=${ROUNDS:-1} timeout 2400 python tools/ab_config.py ${CFG:-C4} base "$@" > $D/ab.jsonl 2> $D/ab.err
cat $D/ab.jsonl; tail -3 $D/ab.err
