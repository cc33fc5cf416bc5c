# panel sweep engine: bitwise tests, then the C4 panel-budget A/B
set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "panel" > gpurun_out/panels_pytest.txt 2>&1
tail -3 gpurun_out/panels_pytest.txt
PDLP_TRACE_SETUP=1 timeout 1200 python tools/panel_sweep.py C4 ${MBS:-40 48 64} > gpurun_out/panel_sweep.jsonl 2> gpurun_out/panel_sweep.err
tail -3 gpurun_out/panel_sweep.err
