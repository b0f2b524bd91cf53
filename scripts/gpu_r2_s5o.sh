# session 5: configs[4] other disorders / seeds at L=250 with the final code; per-level breakdown of one apply at L=150 (ncu launch list with DRAM bytes)
mkdir -p gpurun_out
timeout 900 python scripts/run_config.py 4 21 6 > gpurun_out/s5o_L250_w21_s6.jsonl 2> gpurun_out/s5o_L250_w21_s6.err; cut -c1-330 gpurun_out/s5o_L250_w21_s6.jsonl
timeout 900 python scripts/run_config.py 4 16.5 5 > gpurun_out/s5o_L250_w16_s5.jsonl 2> gpurun_out/s5o_L250_w16_s5.err; cut -c1-330 gpurun_out/s5o_L250_w16_s5.jsonl
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_apply\|k_dense_mv --csv --log-file gpurun_out/s5o_apply150_launches.csv python scripts/prof_kernels.py 150 1 precond > gpurun_out/s5o_ncu.log 2>&1; echo "ncu rc $?"
python scripts/apply_levels.py gpurun_out/s5o_apply150_launches.csv > gpurun_out/s5o_apply_levels_L150.txt 2>&1; head -20 gpurun_out/s5o_apply_levels_L150.txt
