# session 5: persistent ring forward kernel -- parity with every level forced onto it, apply timing at L=150 / 200
mkdir -p gpurun_out
AJ_RING_MIN=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "test_precond_parity and not production" > gpurun_out/s5b_tests_ringall.log 2>&1; echo "tests rc $?"; tail -3 gpurun_out/s5b_tests_ringall.log
for v in "ring:" "noring:AJ_APPLY_RING=0" "ring1m:AJ_RING_MIN=1000000" "ring16m:AJ_RING_MIN=16000000"; do
  name=${v%%:*}; envs=${v#*:}
  env $envs timeout 600 python scripts/prof_kernels.py 150 20 precond > gpurun_out/s5b_apply150_$name.log 2>&1; echo "$name: $(tail -1 gpurun_out/s5b_apply150_$name.log)"
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "production_l48" > gpurun_out/s5b_tests_l48.log 2>&1; echo "tests rc $?"; tail -3 gpurun_out/s5b_tests_l48.log
