# round-2 evidence pass: all GPU tests, smoke, default bench line
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/r2_gpu_tests.log 2>&1; echo "gpu tests rc $?"; tail -15 gpurun_out/r2_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo "smoke rc $?"; tail -2 gpurun_out/r2_smoke.log
timeout 1500 python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo "bench rc $?"; head -c 3000 gpurun_out/r2_bench.json; tail -20 gpurun_out/r2_bench.err
