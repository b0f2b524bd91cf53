# session 5 evidence pass: all GPU tests, smoke, default bench line, bounded ncu launch list, ncu --set full of mid-level apply kernels and the Schur tier kernel (after the parallel A2 phase)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2700 python -m pytest tests -q -m gpu > gpurun_out/s5g_gpu_tests.log 2>&1; echo "gpu tests rc $?"; tail -6 gpurun_out/s5g_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s5g_smoke.log 2>&1; echo "smoke rc $?"; tail -2 gpurun_out/s5g_smoke.log
timeout 1800 python bench.py > gpurun_out/s5g_bench.json 2> gpurun_out/s5g_bench.err; echo "bench rc $?"; head -c 1500 gpurun_out/s5g_bench.json; tail -8 gpurun_out/s5g_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 30000 --csv --log-file gpurun_out/s5g_bench_launches.csv python bench.py --steps 1 --warmup 0 --no-e2e --large "" --big-L 0 --no-cpu-baseline > gpurun_out/s5g_ncu_e.log 2>&1; echo "ncu launches rc $?"
python scripts/ncu_summary.py gpurun_out/s5g_bench_launches.csv 40 > gpurun_out/s5g_bench_launches_summary.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_apply_fwd --launch-skip 5 --launch-count 1 -o gpurun_out/s5g_apply_fwd150_mid python scripts/prof_kernels.py 150 1 precond > gpurun_out/s5g_ncu_c.log 2>&1; echo "ncu fwd rc $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_apply_bwd --launch-skip 185 --launch-count 1 -o gpurun_out/s5g_apply_bwd150_mid python scripts/prof_kernels.py 150 1 precond > gpurun_out/s5g_ncu_b.log 2>&1; echo "ncu bwd rc $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_schur_rows --launch-skip 20 --launch-count 2 -o gpurun_out/s5g_schur150 python scripts/prof_setup.py 150 > gpurun_out/s5g_ncu_d.log 2>&1; echo "ncu schur rc $?"
