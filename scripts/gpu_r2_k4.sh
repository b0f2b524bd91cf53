# round 2: bench line (TMA SpMV, replicated sharded precond), its ncu launch list, W=12 / drop-rule runs, all GPU tests
mkdir -p gpurun_out
export AJ_PARITY_LOG=gpurun_out/r2_parity_errors_k4.jsonl
rm -f $AJ_PARITY_LOG
timeout 1500 python bench.py > gpurun_out/r2_bench_v2.json 2> gpurun_out/r2_bench_v2.err; echo "bench rc $?"; head -c 1500 gpurun_out/r2_bench_v2.json; echo
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_bench_launches.csv python bench.py --steps 1 --warmup 0 --no-e2e --large "" --big-L 0 --no-cpu-baseline > gpurun_out/r2_bench_ncu.log 2>&1; echo "ncu launches rc $?"
bash scripts/gpu_r2_w12.sh
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/r2_gpu_tests_k4.log 2>&1; echo "gpu tests rc $?"; tail -5 gpurun_out/r2_gpu_tests_k4.log
