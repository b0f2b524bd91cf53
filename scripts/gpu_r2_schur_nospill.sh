# round 2: Schur kernels without register spills (launch bounds minBlocks 1): tier bitwise tests + setup timings
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "tiers or precond_parity or inverse_dropping" > gpurun_out/r2_ns_tests.log 2>&1; echo "tests rc $?"; tail -2 gpurun_out/r2_ns_tests.log
for L in 50 100 150 200; do for r in 1 2; do timeout 600 python scripts/prof_setup.py $L 16.5 4 2>&1 | tail -1; done; done > gpurun_out/r2_ns_setup.log; cat gpurun_out/r2_ns_setup.log
