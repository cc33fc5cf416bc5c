cd $GRAFT_REPO_ROOT
D=gpurun_out/${TAG:-r02u}
mkdir -p $D
timeout 900 python tools/setup_trace.py C4 > $D/setup_trace.txt 2>&1; grep -E "upload|create|precondition|plans|offsets" $D/setup_trace.txt
PDLP_UPLOAD_THREADS=0 timeout 900 python tools/setup_trace.py C4 > $D/setup_trace_pageable.txt 2>&1; grep -E "upload|create" $D/setup_trace_pageable.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "transpose or spmv_against or c1_first_100" > $D/pytest.txt 2>&1; tail -2 $D/pytest.txt
