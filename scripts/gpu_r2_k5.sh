# round 2: bench v3 (paper drop rule default, blocked coarse GJ) + ncu captures
mkdir -p gpurun_out
timeout 1800 python bench.py > gpurun_out/r2_bench_v3.json 2> gpurun_out/r2_bench_v3.err; echo "bench rc $?"; head -c 1200 gpurun_out/r2_bench_v3.json; echo; grep -E "step|large|cpu" gpurun_out/r2_bench_v3.err | cut -c1-300
bash scripts/gpu_r2_ncu2.sh
