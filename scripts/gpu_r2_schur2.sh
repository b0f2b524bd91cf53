set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "precond or sqmr or jd_config0 or jd_variants or smoke" > gpurun_out/gpu_tests_b.log 2>&1; echo "tests rc $?"
tail -3 gpurun_out/gpu_tests_b.log
for L in 100 150 200 250; do AJ_VERBOSE=1 timeout 900 python scripts/prof_setup.py $L > gpurun_out/setup${L}_v3.log 2>&1; echo "setup $L rc $?"; tail -1 gpurun_out/setup${L}_v3.log; done
