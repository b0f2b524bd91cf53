# round 2: optimistic W0 Schur tier: bitwise tier tests, setup timings with / without it
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "tiers or precond_parity or inverse_dropping or group_sizes" > gpurun_out/r2_w0_tests.log 2>&1; echo "tests rc $?"; tail -3 gpurun_out/r2_w0_tests.log
for L in 50 150 200; do
  timeout 600 python scripts/prof_setup.py $L 16.5 4 2>&1 | tail -1
  AJ_SCHUR_NO_W0=1 timeout 600 python scripts/prof_setup.py $L 16.5 4 2>&1 | tail -1
done > gpurun_out/r2_w0_setup.log; cat gpurun_out/r2_w0_setup.log
AJ_VERBOSE=1 timeout 600 python scripts/prof_setup.py 200 16.5 3 > gpurun_out/r2_w0_levels200.log 2>&1; grep -c level gpurun_out/r2_w0_levels200.log; sed -n '10p;50p;100p;200p' gpurun_out/r2_w0_levels200.log | cut -c1-330
