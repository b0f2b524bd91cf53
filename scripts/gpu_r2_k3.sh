# round 2: staged apply kernels (bulk-copy factor streams), TMA SpMV v2, replicated sharded preconditioner
mkdir -p gpurun_out
export AJ_PARITY_LOG=gpurun_out/r2_parity_errors.jsonl
rm -f $AJ_PARITY_LOG
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -k "spmv or precond" > gpurun_out/r2_k3_tests.log 2>&1; echo "parity tests rc $?"; tail -3 gpurun_out/r2_k3_tests.log
for L in 50 150 200; do timeout 600 python scripts/prof_kernels.py $L 10 precond2; done > gpurun_out/r2_k3_apply.log 2>&1; cat gpurun_out/r2_k3_apply.log
for L in 250 200; do timeout 300 python scripts/prof_kernels.py $L 20 spmv; done > gpurun_out/r2_k3_spmv.log 2>&1; cat gpurun_out/r2_k3_spmv.log
timeout 2400 python -m pytest tests/test_gpu_sharded.py -q -x > gpurun_out/r2_k3_sharded.log 2>&1; echo "sharded tests rc $?"; tail -5 gpurun_out/r2_k3_sharded.log
