# session 4: concurrent Schur tiers (parity + L=50 / L=150 timings) and the per-phase clock profile of k_schur_rows
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -k "production_l48 or precond_parity or exactness or tier" > gpurun_out/s4e_tests.log 2>&1; echo "tests rc $?"; tail -3 gpurun_out/s4e_tests.log
timeout 300 python scripts/rep_solve.py 1 4 > gpurun_out/s4e_rep50.jsonl 2>&1; tail -1 gpurun_out/s4e_rep50.jsonl
AJ_SCHUR_SERIAL=1 timeout 300 python scripts/rep_solve.py 1 4 > gpurun_out/s4e_rep50_serial.jsonl 2>&1; tail -1 gpurun_out/s4e_rep50_serial.jsonl
timeout 600 python scripts/prof_setup.py 150 > gpurun_out/s4e_setup150.log 2>&1; tail -1 gpurun_out/s4e_setup150.log
AJ_SCHUR_SERIAL=1 timeout 600 python scripts/prof_setup.py 150 > gpurun_out/s4e_setup150_serial.log 2>&1; tail -1 gpurun_out/s4e_setup150_serial.log
AJ_LIB=paper_math_0508111_b200/libaj_schurprof.so timeout 600 python scripts/prof_setup.py 150 > gpurun_out/s4e_schurprof150.log 2>&1; tail -1 gpurun_out/s4e_schurprof150.log
