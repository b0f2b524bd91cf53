# round 2: the paper's drop rule tau_drop = eps/kappa, eps = 1/sqrt(N) vs the auto rule,
# L = 50 .. 250; W=12 with it; repeated L=50 solves (outlier check)
mkdir -p gpurun_out
out=gpurun_out/r2_drop_sweep.jsonl
rm -f $out
timeout 300 python scripts/rep_solve.py 1 15 > gpurun_out/r2_rep50.jsonl 2>&1; tail -3 gpurun_out/r2_rep50.jsonl
AJ_TD=5.657e-4 timeout 300 python scripts/rep_solve.py 1 8 > gpurun_out/r2_rep50_paper.jsonl 2>&1; tail -3 gpurun_out/r2_rep50_paper.jsonl
for L in 150 200 250; do
  td=$(python -c "print(0.2/($L**1.5))")
  AJ_TD=$td AJ_MAX_OUTER=300 timeout 1200 python scripts/run_config.py 2 16.5 2 $L >> $out 2>/dev/null; tail -1 $out | cut -c1-400
done
td=$(python -c "print(0.2/(150**1.5))")
AJ_TD=$td AJ_MAX_OUTER=300 timeout 1200 python scripts/run_config.py 2 16.5 2 150 >> $out 2>/dev/null
AJ_MAX_OUTER=300 timeout 1200 python scripts/run_config.py 2 16.5 2 150 >> $out 2>/dev/null; tail -1 $out | cut -c1-400
AJ_TD=2e-4 AJ_DENSE_CAP=16384 AJ_MAX_OUTER=300 timeout 1200 python scripts/run_config.py 4 12 4 100 >> $out 2> gpurun_out/r2_w12_100_paper.err; tail -1 $out | cut -c1-400
