mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "tiers or precond_parity" > gpurun_out/pt.log 2>&1; tail -2 gpurun_out/pt.log
for L in 50 100 150; do timeout 600 python scripts/prof_kernels.py $L 3 precond 2>&1 | grep "setup"; done
AJ_VERBOSE=1 timeout 600 python scripts/prof_kernels.py 200 3 precond > gpurun_out/v200.log 2>&1; grep -c retry gpurun_out/v200.log; grep "setup L" gpurun_out/v200.log
