# precond parity (incl. Schur tiers) + L=100/150 setup timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "precond" > gpurun_out/pt.log 2>&1; tail -3 gpurun_out/pt.log
AJ_VERBOSE=1 timeout 300 python scripts/prof_kernels.py 100 3 precond > gpurun_out/v100.log 2>&1; tail -2 gpurun_out/v100.log
AJ_VERBOSE=1 timeout 600 python scripts/prof_kernels.py 150 3 precond > gpurun_out/v150.log 2>&1; tail -2 gpurun_out/v150.log
