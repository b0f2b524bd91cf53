# session 4: ncu launch list (per-launch durations, in order) of one L=50 setup
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s4_setup50_launches.csv python scripts/prof_setup.py 50 16.5 1 > gpurun_out/s4_setup50_ncu.log 2>&1; echo "ncu rc $?"
python scripts/ncu_summary.py gpurun_out/s4_setup50_launches.csv 40
