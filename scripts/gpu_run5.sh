mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "precond or coarse or jd_config1 or jd_variants" > gpurun_out/pt.log 2>&1; tail -2 gpurun_out/pt.log
AJ_VERBOSE=1 timeout 300 python scripts/prof_kernels.py 50 3 precond 1 2>&1 | grep "coarse\|setup L"
AJ_VERBOSE=1 timeout 300 python scripts/prof_kernels.py 100 3 precond 2>&1 | grep "coarse\|setup L"
timeout 300 python scripts/run_config.py 1 2>&1 | tail -1 | cut -c1-200
