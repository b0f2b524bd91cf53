# configs[3] and configs[4] (W=16.5 seed 4, W=21 seed 6) with the library defaults
mkdir -p gpurun_out
: > gpurun_out/large.jsonl
timeout 600 python scripts/run_config.py 3 > gpurun_out/l200.log 2>&1; tail -1 gpurun_out/l200.log >> gpurun_out/large.jsonl
timeout 900 python scripts/run_config.py 4 > gpurun_out/l250.log 2>&1; tail -1 gpurun_out/l250.log >> gpurun_out/large.jsonl
timeout 900 python scripts/run_config.py 4 21.0 6 > gpurun_out/l250w21.log 2>&1; tail -1 gpurun_out/l250w21.log >> gpurun_out/large.jsonl
cut -c1-260 gpurun_out/large.jsonl
