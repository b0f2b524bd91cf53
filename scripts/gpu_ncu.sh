# ncu --set full captures: level-0 and a mid-level forward apply kernel at L=150, the SpMV at L=250
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_apply_fwd" --launch-skip 0 --launch-count 1 -o gpurun_out/fwd0_150 python scripts/prof_kernels.py 150 1 precond > gpurun_out/ncu1.log 2>&1; echo "fwd0 $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_apply_bwd" --launch-skip 120 --launch-count 1 -o gpurun_out/bwdmid_150 python scripts/prof_kernels.py 150 1 precond > gpurun_out/ncu2.log 2>&1; echo "bwd $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_spmv" --launch-skip 2 --launch-count 1 -o gpurun_out/spmv250 python scripts/prof_kernels.py 250 3 spmv > gpurun_out/ncu3.log 2>&1; echo "spmv $?"
