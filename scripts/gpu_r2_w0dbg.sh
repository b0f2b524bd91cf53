mkdir -p gpurun_out
AJ_VERBOSE=1 timeout 300 python scripts/prof_setup.py 50 16.5 4 > gpurun_out/r2_w0dbg_50.log 2>&1; grep -E "level (0|5|10|20|30) " gpurun_out/r2_w0dbg_50.log | cut -c1-300; tail -1 gpurun_out/r2_w0dbg_50.log
AJ_VERBOSE=1 timeout 600 python scripts/prof_setup.py 100 16.5 4 > gpurun_out/r2_w0dbg_100.log 2>&1; tail -4 gpurun_out/r2_w0dbg_100.log | cut -c1-300
timeout 1200 compute-sanitizer --tool memcheck --print-limit 5 python scripts/prof_setup.py 100 16.5 4 > gpurun_out/r2_w0dbg_san.log 2>&1; head -60 gpurun_out/r2_w0dbg_san.log
