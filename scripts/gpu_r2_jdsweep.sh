# round 2: JD inner settings with the paper's drop rule (inner_tol x inner_max) at L=50 and L=150
mkdir -p gpurun_out
out=gpurun_out/r2_jd_sweep.jsonl
rm -f $out
for L in 50 150; do
 for tol in 3e-3 1e-2 3e-2 1e-1; do
  for im in 60 150; do
   AJ_INNER_TOL=$tol AJ_INNER_MAX=$im AJ_MAX_OUTER=400 timeout 600 python scripts/run_config.py 1 16.5 1 $L >> $out 2>/dev/null
   tail -1 $out | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['L'], d['env'].get('AJ_INNER_TOL'), d['env'].get('AJ_INNER_MAX'), round(d.get('wall_s',0),3), d.get('setup_ms'), d.get('solve_ms'), d.get('outer'), d.get('inner'), d.get('error','')[:80])"
  done
 done
done
