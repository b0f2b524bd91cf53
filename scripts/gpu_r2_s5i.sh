# session 5: missed-eigenvalue safeguard in JD -- the sharded small test, how often it triggers at the configs (verbose log), timing impact; coarse cutover at L=50; bounded ncu launch list of the bench command
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_sharded.py -q -x -k "small_matches_dense or two_ranks_config1" > gpurun_out/s5i_tests_sharded.log 2>&1; echo "tests rc $?"; tail -3 gpurun_out/s5i_tests_sharded.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "jd_config0 or jd_variants or jd_config1" > gpurun_out/s5i_tests_jd.log 2>&1; echo "tests rc $?"; tail -3 gpurun_out/s5i_tests_jd.log
for c in 1 2 3; do
  timeout 900 python scripts/run_config.py $c > gpurun_out/s5i_cfg$c.jsonl 2> gpurun_out/s5i_cfg$c.err; echo "cfg $c: $(cut -c1-260 gpurun_out/s5i_cfg$c.jsonl)"; grep -c "continuing" gpurun_out/s5i_cfg$c.err
done
timeout 900 python scripts/run_config.py 4 16.5 4 > gpurun_out/s5i_cfg4.jsonl 2> gpurun_out/s5i_cfg4.err; echo "cfg 4: $(cut -c1-260 gpurun_out/s5i_cfg4.jsonl)"; grep -c "continuing" gpurun_out/s5i_cfg4.err
for nc in 1024 1536 2048 3072; do
  AJ_NCOARSE=$nc timeout 300 python scripts/rep_solve.py 1 4 > gpurun_out/s5h_rep50_nc$nc.jsonl 2>&1; echo "nc=$nc: $(tail -1 gpurun_out/s5h_rep50_nc$nc.jsonl)"
done
timeout 2400 ncu --metrics gpu__time_duration.sum --clock-control none -c 30000 --csv --log-file gpurun_out/s5g_bench_launches.csv python bench.py --steps 1 --warmup 0 --no-e2e --large "" --big-L 0 --no-cpu-baseline > gpurun_out/s5g_ncu_e.log 2>&1; echo "ncu launches rc $?"
python scripts/ncu_summary.py gpurun_out/s5g_bench_launches.csv 40 > gpurun_out/s5g_bench_launches_summary.txt 2>&1; head -5 gpurun_out/s5g_bench_launches_summary.txt
