# tau_strong sweep at L=100 / 150 (R17): setup/solve/levels
mkdir -p gpurun_out
for ts in 0.035 0.05; do AJ_TS=$ts AJ_MAX_OUTER=200 timeout 400 python scripts/run_config.py 2 > gpurun_out/sw100_$ts.log 2>&1; echo "L100 ts=$ts"; tail -1 gpurun_out/sw100_$ts.log | cut -c1-330; done
for ts in 0.02 0.035; do AJ_TS=$ts AJ_MAX_OUTER=200 timeout 600 python scripts/run_config.py 2 16.5 2 150 > gpurun_out/sw150_$ts.log 2>&1; echo "L150 ts=$ts"; tail -1 gpurun_out/sw150_$ts.log | cut -c1-330; done
