mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "sqmr or jd_config0 or jd_variants or jd_config1 or host" > gpurun_out/pt.log 2>&1; tail -2 gpurun_out/pt.log
for c in 1 1 2; do timeout 300 python scripts/run_config.py $c 2>&1 | tail -1 | cut -c1-220; done
