set -x
mkdir -p gpurun_out
# level ~40 of L=150: launches of k_schur_rows (tiers run in sequence per level)
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_schur_rows" --launch-skip 120 --launch-count 4 -o gpurun_out/schur_rows150 python scripts/prof_setup.py 150 > gpurun_out/ncu_schur_rows.log 2>&1; echo "ncu rc $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/setup150_launches_v2.csv python scripts/prof_setup.py 150 > gpurun_out/setup150_ncu_v2.log 2>&1; echo "ncu list rc $?"
python scripts/ncu_summary.py gpurun_out/setup150_launches_v2.csv 30 > gpurun_out/setup150_summary_v2.txt 2>&1
