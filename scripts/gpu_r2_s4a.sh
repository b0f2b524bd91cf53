# session 4: level logs at L=50 (configs[1]) and W=12 L=100, for the dense-coarse work
mkdir -p gpurun_out
AJ_VERBOSE=1 timeout 300 python scripts/rep_solve.py 1 2 > gpurun_out/s4_levels_L50.log 2>&1; tail -2 gpurun_out/s4_levels_L50.log
AJ_VERBOSE=1 AJ_DENSE_CAP=16384 AJ_MAX_OUTER=300 timeout 1200 python scripts/run_config.py 4 12 4 100 > gpurun_out/s4_w12_L100.log 2>&1; tail -c 800 gpurun_out/s4_w12_L100.log
