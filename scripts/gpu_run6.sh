mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "precond" > gpurun_out/pt.log 2>&1; tail -2 gpurun_out/pt.log
for L in 50 100 150; do timeout 600 python scripts/prof_kernels.py $L 3 precond 2>&1 | grep "setup"; done
for i in 1 2; do timeout 300 python scripts/run_config.py 1 2>&1 | tail -1 | cut -c1-200; done
