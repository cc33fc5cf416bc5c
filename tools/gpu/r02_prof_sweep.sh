# ncu --set full of the C4 panel SpMV over K: the committed round-1 kernel (variant orig) and the current one
cd $GRAFT_REPO_ROOT
D=gpurun_out/${TAG:-r02k}
mkdir -p $D
NCU_SOLVE=0 PDLP_LIB=paper_2311_12180_b200/lib/variants/orig.so timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"sweep_spmv" -c 3 -o $D/orig python tools/ncu_kernels.py C4 2 > $D/orig.log 2>&1; tail -2 $D/orig.log
NCU_SOLVE=0 PDLP_LIB=paper_2311_12180_b200/lib/variants/${NEWV:-r128}.so timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"sweep_kernel" -c 1 -o $D/new python tools/ncu_kernels.py C4 2 > $D/new.log 2>&1; tail -2 $D/new.log
