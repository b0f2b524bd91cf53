# session 5: entry-tiled apply kernels -- parity (all levels forced), apply timing at L=150 and L=200
mkdir -p gpurun_out
AJ_TILE_MIN=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "test_precond_parity and not production" > gpurun_out/s5d_tests_tileall.log 2>&1; echo "tests rc $?"; tail -3 gpurun_out/s5d_tests_tileall.log
for v in "tile:" "notile:AJ_APPLY_TILE=0" "tile1m:AJ_TILE_MIN=1000000" "tile256k:AJ_TILE_MIN=262144" "tile16m:AJ_TILE_MIN=16000000"; do
  name=${v%%:*}; envs=${v#*:}
  env $envs timeout 600 python scripts/prof_kernels.py 150 20 precond > gpurun_out/s5d_apply150_$name.log 2>&1; echo "$name: $(tail -1 gpurun_out/s5d_apply150_$name.log)"
done
for v in "tile:" "notile:AJ_APPLY_TILE=0"; do
  name=${v%%:*}; envs=${v#*:}
  env $envs timeout 600 python scripts/prof_kernels.py 200 10 precond > gpurun_out/s5d_apply200_$name.log 2>&1; echo "L200 $name: $(tail -1 gpurun_out/s5d_apply200_$name.log)"
done
