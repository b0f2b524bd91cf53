mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "precond or sqmr or jd_config1" > gpurun_out/pt.log 2>&1; tail -2 gpurun_out/pt.log
for L in 50 100 150 200; do timeout 600 python scripts/prof_kernels.py $L 10 precond 2>&1 | grep "apply"; done
