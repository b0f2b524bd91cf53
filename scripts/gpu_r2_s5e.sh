# session 5: tile kernels parity after the pre-wait fix; dependency-free timing diagnostic (pdl_wait compiled out); parallel A2 phase of the Schur kernel (parity + setup time)
mkdir -p gpurun_out
AJ_TILE_MIN=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "test_precond_parity and not production" > gpurun_out/s5e_tests_tileall.log 2>&1; echo "tests rc $?"; tail -3 gpurun_out/s5e_tests_tileall.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "test_precond_parity and not production" > gpurun_out/s5e_tests_default.log 2>&1; echo "tests rc $?"; tail -3 gpurun_out/s5e_tests_default.log
for v in "nowait_tile:AJ_LIB=paper_math_0508111_b200/libaj_nowait.so" "nowait_notile:AJ_APPLY_TILE=0 AJ_LIB=paper_math_0508111_b200/libaj_nowait.so" "nowait_tile256k:AJ_TILE_MIN=262144 AJ_LIB=paper_math_0508111_b200/libaj_nowait.so"; do
  name=${v%%:*}; envs=${v#*:}
  env $envs timeout 600 python scripts/prof_kernels.py 150 20 precond > gpurun_out/s5e_apply150_$name.log 2>&1; echo "$name: $(tail -1 gpurun_out/s5e_apply150_$name.log)"
done
timeout 600 python scripts/prof_setup.py 150 > gpurun_out/s5e_setup150.log 2>&1; tail -1 gpurun_out/s5e_setup150.log
timeout 300 python scripts/rep_solve.py 1 4 > gpurun_out/s5e_rep50.jsonl 2>&1; tail -1 gpurun_out/s5e_rep50.jsonl
