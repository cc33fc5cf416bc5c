cd $GRAFT_REPO_ROOT
D=gpurun_out/${TAG:-r02w}
mkdir -p $D
PDLP_LIB=$GRAFT_REPO_ROOT/paper_2311_12180_b200/lib/variants/pipe4.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "column_panel" > $D/pytest_pipe4.txt 2>&1; tail -2 $D/pytest_pipe4.txt
AB_ROUNDS=2 timeout 2400 python tools/ab_config.py C4 base "pipe5:x:" "pipe4:x:" > $D/ab.jsonl 2> $D/ab.err; cat $D/ab.jsonl; tail -3 $D/ab.err
