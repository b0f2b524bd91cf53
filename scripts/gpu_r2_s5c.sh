# session 5: ring kernels, forward + backward: parity (all levels forced), timing of the variants at L=150
mkdir -p gpurun_out
AJ_APPLY_RING=1 AJ_RING_MIN=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "test_precond_parity and not production" > gpurun_out/s5c_tests_ringall.log 2>&1; echo "tests rc $?"; tail -3 gpurun_out/s5c_tests_ringall.log
for v in "both:AJ_APPLY_RING=1" "fwdonly:AJ_APPLY_RING=1 AJ_APPLY_RING_BWD=0" "both8:AJ_APPLY_RING=1 AJ_LIB=paper_math_0508111_b200/libaj_ring8.so" "bothbig:AJ_APPLY_RING=1 AJ_LIB=paper_math_0508111_b200/libaj_ringbig.so" "bothbig1m:AJ_APPLY_RING=1 AJ_RING_MIN=1000000 AJ_LIB=paper_math_0508111_b200/libaj_ringbig.so"; do
  name=${v%%:*}; envs=${v#*:}
  env $envs timeout 600 python scripts/prof_kernels.py 150 20 precond > gpurun_out/s5c_apply150_$name.log 2>&1; echo "$name: $(tail -1 gpurun_out/s5c_apply150_$name.log)"
done
