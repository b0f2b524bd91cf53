# session 4: optimistic Schur tier -- parity with the tier off / forced, then timings
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -k "production_l48 or precond_parity or exactness" > gpurun_out/s4c_tests.log 2>&1; echo "tests rc $?"; tail -3 gpurun_out/s4c_tests.log
timeout 300 python scripts/rep_solve.py 1 4 > gpurun_out/s4c_rep50.jsonl 2>&1; tail -2 gpurun_out/s4c_rep50.jsonl
AJ_SCHUR_OPT=0 timeout 300 python scripts/rep_solve.py 1 4 > gpurun_out/s4c_rep50_noopt.jsonl 2>&1; tail -1 gpurun_out/s4c_rep50_noopt.jsonl
AJ_VERBOSE=1 timeout 600 python scripts/prof_setup.py 150 > gpurun_out/s4c_setup150.log 2>&1; tail -1 gpurun_out/s4c_setup150.log
AJ_SCHUR_OPT=0 timeout 600 python scripts/prof_setup.py 150 > gpurun_out/s4c_setup150_noopt.log 2>&1; tail -1 gpurun_out/s4c_setup150_noopt.log
AJ_VERBOSE=1 timeout 600 python scripts/prof_setup.py 200 16.5 3 > gpurun_out/s4c_setup200.log 2>&1; tail -1 gpurun_out/s4c_setup200.log
