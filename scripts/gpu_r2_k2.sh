# round 2: SpMV variants (balanced one-wave / tiled / TMA) + apply ncu captures
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "spmv" > gpurun_out/r2_k2_tests.log 2>&1; echo "tests rc $?"; tail -3 gpurun_out/r2_k2_tests.log
for L in 250 200 100 50; do timeout 300 python scripts/prof_kernels.py $L 20 spmv; done > gpurun_out/r2_k2_spmv.log 2>&1; cat gpurun_out/r2_k2_spmv.log
AJ_SPMV_PATH=bal timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_spmv2_bal --launch-skip 2 --launch-count 1 -o gpurun_out/r2_spmv_bal250 python scripts/prof_kernels.py 250 3 spmv > gpurun_out/r2_k2_ncu1.log 2>&1; echo "ncu1 rc $?"
AJ_SPMV_PATH=tma timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_spmv_tma --launch-skip 2 --launch-count 1 -o gpurun_out/r2_spmv_tma250b python scripts/prof_kernels.py 250 3 spmv > gpurun_out/r2_k2_ncu2.log 2>&1; echo "ncu2 rc $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_apply_bwd --launch-skip 300 --launch-count 3 -o gpurun_out/r2_apply_bwd150 python scripts/prof_kernels.py 150 2 precond > gpurun_out/r2_k2_ncu3.log 2>&1; echo "ncu3 rc $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_apply_fwd --launch-skip 200 --launch-count 3 -o gpurun_out/r2_apply_fwd150 python scripts/prof_kernels.py 150 2 precond > gpurun_out/r2_k2_ncu4.log 2>&1; echo "ncu4 rc $?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_apply150_launches.csv python scripts/prof_kernels.py 150 1 precond > gpurun_out/r2_k2_ncu5.log 2>&1; echo "ncu5 rc $?"
