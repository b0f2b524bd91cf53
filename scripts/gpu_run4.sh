# W=12 L=100: level row cap 300 + dense coarse up to 12288
mkdir -p gpurun_out
AJ_ROWCAP=300 AJ_DENSE_CAP=12288 AJ_MAX_OUTER=300 timeout 600 python scripts/run_config.py 4 12.0 5 100 > gpurun_out/w12_100_dc.log 2>&1; tail -1 gpurun_out/w12_100_dc.log | cut -c1-400
