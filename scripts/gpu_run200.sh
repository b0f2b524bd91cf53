# configs[3] (L=200) and configs[4] (L=250, W=16.5) on one GPU
mkdir -p gpurun_out
AJ_MAX_OUTER=250 timeout 900 python scripts/run_config.py 3 > gpurun_out/rc200.log 2>&1; tail -1 gpurun_out/rc200.log | cut -c1-700
AJ_VERBOSE=1 AJ_MAX_OUTER=250 timeout 1500 python scripts/run_config.py 4 > gpurun_out/rc250.log 2>&1; tail -1 gpurun_out/rc250.log | cut -c1-700
