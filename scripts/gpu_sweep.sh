# experimental tau_strong depth growth (AJ_TS_ALPHA) at L=100 / 150
mkdir -p gpurun_out
for a in 0.15 0.3; do AJ_TS_ALPHA=$a AJ_MAX_OUTER=150 timeout 400 python scripts/run_config.py 2 > gpurun_out/sa100_$a.log 2>&1; echo "L100 a=$a"; tail -1 gpurun_out/sa100_$a.log | cut -c1-300; done
for a in 0.15 0.3; do AJ_TS_ALPHA=$a AJ_MAX_OUTER=150 timeout 600 python scripts/run_config.py 2 16.5 2 150 > gpurun_out/sa150_$a.log 2>&1; echo "L150 a=$a"; tail -1 gpurun_out/sa150_$a.log | cut -c1-300; done
