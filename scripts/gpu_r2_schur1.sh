set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?"
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "precond or sqmr or jd_config0 or jd_variants or disorder" > gpurun_out/gpu_tests_a.log 2>&1; echo "tests rc $?"
for L in 100 150 200 250; do AJ_VERBOSE=1 timeout 900 python scripts/prof_setup.py $L > gpurun_out/setup${L}_v2.log 2>&1; echo "setup $L rc $?"; tail -1 gpurun_out/setup${L}_v2.log; done
