# round 2: TMA SpMV + batched apply gathers: parity, timings, one ncu capture of the TMA SpMV
mkdir -p gpurun_out
export AJ_PARITY_LOG=gpurun_out/r2_parity_errors.jsonl
rm -f $AJ_PARITY_LOG
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "spmv or precond" > gpurun_out/r2_k1_tests.log 2>&1; echo "tests rc $?"; tail -3 gpurun_out/r2_k1_tests.log
timeout 300 python scripts/prof_kernels.py 250 20 spmv > gpurun_out/r2_k1_spmv.log 2>&1; cat gpurun_out/r2_k1_spmv.log
timeout 300 python scripts/prof_kernels.py 200 20 spmv >> gpurun_out/r2_k1_spmv.log 2>&1; tail -2 gpurun_out/r2_k1_spmv.log
timeout 300 python scripts/prof_kernels.py 100 50 spmv >> gpurun_out/r2_k1_spmv.log 2>&1; tail -2 gpurun_out/r2_k1_spmv.log
timeout 600 python scripts/prof_kernels.py 150 10 precond > gpurun_out/r2_k1_apply.log 2>&1; cat gpurun_out/r2_k1_apply.log
timeout 600 python scripts/prof_kernels.py 200 10 precond >> gpurun_out/r2_k1_apply.log 2>&1; tail -2 gpurun_out/r2_k1_apply.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_spmv_tma --launch-skip 2 --launch-count 1 -o gpurun_out/r2_spmv_tma250 python scripts/prof_kernels.py 250 3 spmv > gpurun_out/r2_k1_ncu.log 2>&1; echo "ncu rc $?"
