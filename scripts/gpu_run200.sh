# configs[3] (L=200) on one GPU with setup verbosity
mkdir -p gpurun_out
AJ_VERBOSE=1 AJ_MAX_OUTER=250 timeout 1500 python scripts/run_config.py 3 > gpurun_out/rc200.log 2>&1; tail -1 gpurun_out/rc200.log | cut -c1-600
