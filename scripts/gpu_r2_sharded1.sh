set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_gpu_sharded.py -x -q -k "not config1" > gpurun_out/gpu_sharded_a.log 2>&1; echo "sharded tests rc $?"
tail -30 gpurun_out/gpu_sharded_a.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "slab or spmv" > gpurun_out/gpu_tests_slab.log 2>&1; echo "slab tests rc $?"
tail -3 gpurun_out/gpu_tests_slab.log
