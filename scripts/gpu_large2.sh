# configs[4] robustness: more seeds at L=250 (W=16.5 seeds 5, 6; W=21 seed 4)
mkdir -p gpurun_out
: > gpurun_out/large2.jsonl
for ws in "16.5 5" "16.5 6" "21.0 4"; do set -- $ws
  timeout 900 python scripts/run_config.py 4 $1 $2 > gpurun_out/l250s.log 2>&1; tail -1 gpurun_out/l250s.log >> gpurun_out/large2.jsonl
done
cut -c1-250 gpurun_out/large2.jsonl
