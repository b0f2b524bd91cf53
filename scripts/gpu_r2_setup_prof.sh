set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc; lscpu | grep -E "Model name|^CPU\(s\)|Thread"
AJ_VERBOSE=1 timeout 600 python scripts/prof_setup.py 150 > gpurun_out/setup150_verbose.log 2>&1; echo "verbose rc $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/setup150_launches.csv python scripts/prof_setup.py 150 > gpurun_out/setup150_ncu.log 2>&1; echo "ncu rc $?"
python scripts/ncu_summary.py gpurun_out/setup150_launches.csv 40 > gpurun_out/setup150_summary.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_schur" --launch-skip 40 --launch-count 1 -o gpurun_out/schur150 python scripts/prof_setup.py 150 > gpurun_out/ncu_schur.log 2>&1; echo "ncu full rc $?"
