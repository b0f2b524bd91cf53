# session 5: per-level setup logs with the final code (L=250 and L=50)
mkdir -p gpurun_out
AJ_VERBOSE=1 timeout 600 python scripts/prof_setup.py 250 > gpurun_out/s5p_setup_levels_L250.log 2>&1; tail -2 gpurun_out/s5p_setup_levels_L250.log | cut -c1-200
AJ_VERBOSE=1 timeout 600 python scripts/prof_setup.py 50 16.5 1 > gpurun_out/s5p_setup_levels_L50.log 2>&1; tail -2 gpurun_out/s5p_setup_levels_L50.log | cut -c1-200
