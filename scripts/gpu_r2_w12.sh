# round 2: configs[4] W=12 (dense coarse cap), and the paper's drop rule (eps = 1/sqrt(N), l.1093) vs the auto rule
mkdir -p gpurun_out
out=gpurun_out/r2_w12_drop.jsonl
rm -f $out
AJ_VERBOSE=0 AJ_MAX_OUTER=300 timeout 900 python scripts/run_config.py 4 12 4 100 >> $out 2> gpurun_out/r2_w12_100_default.err; tail -1 $out
AJ_DENSE_CAP=16384 AJ_MAX_OUTER=300 timeout 1200 python scripts/run_config.py 4 12 4 100 >> $out 2> gpurun_out/r2_w12_100_cap.err; tail -1 $out
# paper: drop tolerance eps/kappa with eps = 1/sqrt(N) = 1e-3 at L=100, aggressive dropping with tau = eps (and tau = 0.1, the paper's example)
AJ_TD=2e-4 AJ_MAX_OUTER=300 timeout 900 python scripts/run_config.py 2 16.5 2 100 >> $out 2>/dev/null; tail -1 $out
AJ_TD=2e-4 AJ_TINV=1e-3 AJ_MAX_OUTER=300 timeout 900 python scripts/run_config.py 2 16.5 2 100 >> $out 2>/dev/null; tail -1 $out
AJ_TD=2e-4 AJ_TINV=0.1 AJ_MAX_OUTER=300 timeout 900 python scripts/run_config.py 2 16.5 2 100 >> $out 2>/dev/null; tail -1 $out
AJ_TINV=0.1 AJ_MAX_OUTER=300 timeout 900 python scripts/run_config.py 2 16.5 2 100 >> $out 2>/dev/null; tail -1 $out
AJ_MAX_OUTER=300 timeout 900 python scripts/run_config.py 2 16.5 2 100 >> $out 2>/dev/null; tail -1 $out
