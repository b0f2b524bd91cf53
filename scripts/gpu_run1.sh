# ad-hoc GPU check: parity of the preconditioner + setup/solve timings at L=50/100/150
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "precond or jd" > gpurun_out/pt.log 2>&1; tail -3 gpurun_out/pt.log
AJ_VERBOSE=1 timeout 300 python scripts/prof_kernels.py 100 3 precond > gpurun_out/v100.log 2>&1; tail -2 gpurun_out/v100.log
for c in 1 2; do timeout 300 python scripts/run_config.py $c > gpurun_out/rc$c.log 2>&1; tail -1 gpurun_out/rc$c.log | cut -c1-400; done
AJ_MAX_OUTER=300 timeout 600 python scripts/run_config.py 2 16.5 2 150 > gpurun_out/rc150.log 2>&1; tail -1 gpurun_out/rc150.log | cut -c1-400
