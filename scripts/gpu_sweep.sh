# tau_drop exponent: 2e-3 (50/L)^p for p = 1.5 and 1.0 at L=150 / 200 (tau_strong, tau_virtual follow)
mkdir -p gpurun_out
for L in 150 200; do for pw in 1.5 1.0; do
td=$(python -c "print(2e-3*(50/$L)**$pw)")
AJ_TD=$td AJ_MAX_OUTER=150 timeout 600 python scripts/run_config.py 3 16.5 3 $L > gpurun_out/sw.log 2>&1; echo "L=$L p=$pw td=$td $(tail -1 gpurun_out/sw.log | python -c 'import sys,json
try:
  d=json.loads(sys.stdin.read()); print(round(d["wall_s"],2), round(d["setup_ms"]), round(d["solve_ms"]), d["outer"], d["inner"], d["levels"], round(d["nnzL_per_site"],1))
except Exception as e: print("fail")')"; done; done
