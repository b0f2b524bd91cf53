# round 2: blocked Gauss-Jordan coarse inverse: parity, setup timings, W=12 at L=100 with the paper's drop rule
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "coarse or l48 or exactness or precond_parity" > gpurun_out/r2_gj_tests.log 2>&1; echo "tests rc $?"; tail -3 gpurun_out/r2_gj_tests.log
timeout 300 python scripts/rep_solve.py 1 5 > gpurun_out/r2_gj_rep50.jsonl 2>&1; tail -2 gpurun_out/r2_gj_rep50.jsonl
AJ_TD=5.657e-4 timeout 300 python scripts/rep_solve.py 1 5 > gpurun_out/r2_gj_rep50_paper.jsonl 2>&1; tail -2 gpurun_out/r2_gj_rep50_paper.jsonl
AJ_TD=2e-4 AJ_DENSE_CAP=16384 AJ_MAX_OUTER=300 timeout 1200 python scripts/run_config.py 4 12 4 100 > gpurun_out/r2_gj_w12.jsonl 2> gpurun_out/r2_gj_w12.err; cut -c1-600 gpurun_out/r2_gj_w12.jsonl
