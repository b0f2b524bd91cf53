# session 5: W=12 at M=130 with the final code and DEFAULT parameters (no environment overrides)
mkdir -p gpurun_out
AJ_MAX_OUTER=300 timeout 1500 python scripts/run_config.py 4 12 4 130 > gpurun_out/s5r_w12_L130.jsonl 2> gpurun_out/s5r_w12_L130.err; cut -c1-500 gpurun_out/s5r_w12_L130.jsonl
