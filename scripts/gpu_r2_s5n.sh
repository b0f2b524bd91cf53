# session 5 final evidence pass: all GPU tests, smoke, default bench line
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 3000 python -m pytest tests -q -m gpu > gpurun_out/s5n_gpu_tests.log 2>&1; echo "gpu tests rc $?"; tail -6 gpurun_out/s5n_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s5n_smoke.log 2>&1; echo "smoke rc $?"; tail -2 gpurun_out/s5n_smoke.log
timeout 1800 python bench.py > gpurun_out/s5n_bench.json 2> gpurun_out/s5n_bench.err; echo "bench rc $?"; head -c 600 gpurun_out/s5n_bench.json; echo; tail -6 gpurun_out/s5n_bench.err | cut -c1-400
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/s5n_bench_ref.json 2> gpurun_out/s5n_bench_ref.err; echo "ref rc $?"; head -c 600 gpurun_out/s5n_bench_ref.json
