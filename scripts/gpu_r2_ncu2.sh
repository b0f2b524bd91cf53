# round 2: ncu --set full of the final TMA SpMV (L=250), mid-level apply kernels (L=150 level ~5),
# a Schur-tier setup kernel (L=150), and a bounded launch list of the bench command
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_spmv_tma --launch-skip 2 --launch-count 1 -o gpurun_out/r2_spmv_tma250c python scripts/prof_kernels.py 250 3 spmv > gpurun_out/r2_ncu2_a.log 2>&1; echo "ncu spmv rc $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_apply_bwd --launch-skip 123 --launch-count 1 -o gpurun_out/r2_apply_bwd150_mid python scripts/prof_kernels.py 150 1 precond > gpurun_out/r2_ncu2_b.log 2>&1; echo "ncu bwd rc $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_apply_fwd --launch-skip 5 --launch-count 1 -o gpurun_out/r2_apply_fwd150_mid python scripts/prof_kernels.py 150 1 precond > gpurun_out/r2_ncu2_c.log 2>&1; echo "ncu fwd rc $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_schur_rows --launch-skip 20 --launch-count 2 -o gpurun_out/r2_schur150 python scripts/prof_setup.py 150 > gpurun_out/r2_ncu2_d.log 2>&1; echo "ncu schur rc $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 30000 --csv --log-file gpurun_out/r2_bench_launches2.csv python bench.py --steps 1 --warmup 0 --no-e2e --large "" --big-L 0 --no-cpu-baseline > gpurun_out/r2_ncu2_e.log 2>&1; echo "ncu launches rc $?"
python scripts/ncu_summary.py gpurun_out/r2_bench_launches2.csv 40 > gpurun_out/r2_bench_launches_summary.txt 2>&1
