#!/bin/bash
run() { python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --big-L 0 "$@" 2>/dev/null | python -c "
import json,sys
try:
  d=json.loads(sys.stdin.read()); j=d['jd']
  print('$*', 'step %.1f ms'%d['ms_per_step'], 'setup %.1f'%j['setup_ms'], 'solve %.1f'%j['solve_ms'], 'outer', j['outer'], 'inner', j['inner_total'], 'levels', j['levels'], flush=True)
except Exception as e: print('$*', 'FAILED', e)" ; }
run --inner-tol 0.01
run --inner-tol 0.003
run --inner-tol 0.001
run --inner-tol 0.01 --inner-max 100
run --inner-tol 0.01 --switch-tol 1e-4
run --inner-tol 0.01 --jmin 8 --jmax 30
run --inner-tol 0.01 --tau-drop 1e-3
