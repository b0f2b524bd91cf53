# session 5: Schur kernel -- warp-ballot work-list compaction and rank sort of the short L-row / virtual-term lists: parity + setup timings
mkdir -p gpurun_out
timeout 600 python scripts/prof_setup.py 150 > gpurun_out/s5k_setup150.log 2>&1; tail -1 gpurun_out/s5k_setup150.log
timeout 300 python scripts/rep_solve.py 1 4 > gpurun_out/s5k_rep50.jsonl 2>&1; tail -1 gpurun_out/s5k_rep50.jsonl
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -k "precond" > gpurun_out/s5k_tests_precond.log 2>&1; echo "tests rc $?"; tail -3 gpurun_out/s5k_tests_precond.log
timeout 600 python scripts/run_config.py 3 > gpurun_out/s5k_cfg3.jsonl 2> gpurun_out/s5k_cfg3.err; cut -c1-260 gpurun_out/s5k_cfg3.jsonl
