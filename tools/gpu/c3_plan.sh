cd $GRAFT_REPO_ROOT
PDLP_TRACE_SETUP=1 timeout 300 python -c "
from paper_2311_12180_b200 import Solver, SolverParams, generators
for c in ('C2','C3'):
    s = Solver(generators.config(c), SolverParams()); s.close()
" 2>&1 | grep tiles
export PDLP_GRAPH=0 PDLP_ITER_LIMIT=64
timeout 900 ncu --set full --cache-control none --clock-control none -k regex:"dual_kernel|primal_kernel|spmv_kernel" -s 30 -c 3 -o gpurun_out/prof_c3 python tools/profile_c2.py C3 > gpurun_out/prof_c3.log 2>&1
tail -1 gpurun_out/prof_c3.log
