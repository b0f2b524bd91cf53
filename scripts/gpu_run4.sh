# inner_max 100 / 150 at W=16.5, L=50/100/200; W=12 L=100 with row cap 300 and dense_cap 10000
mkdir -p gpurun_out
for im in 100 150; do for c in 1 2 3; do AJ_INNER_MAX=$im AJ_MAX_OUTER=300 timeout 400 python scripts/run_config.py $c > gpurun_out/im${im}_c$c.log 2>&1; echo "inner_max=$im config=$c: $(tail -1 gpurun_out/im${im}_c$c.log | cut -c1-200)"; done; done
