#!/bin/bash
# parameter sweep of the L=50 step (GPU): prints one summary line per setting
run() { python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --big-L 0 "$@" 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); j=d['jd']
print('$*', 'step %.1f ms'%d['ms_per_step'], 'setup %.1f'%j['setup_ms'], 'solve %.1f'%j['solve_ms'], 'outer', j['outer'], 'inner', j['inner_total'], 'levels', j['levels'], 'coarse', j['coarse_n'])" ; }
run
run --tau-strong 0.05
run --tau-strong 0.1
run --tau-drop 4e-3 --tau-strong 0.04
run --tau-drop 1e-3 --tau-strong 0.02
run --inner-tol 0.01
run --inner-tol 0.3
run --inner-max 20
run --jmin 5 --jmax 15
run --switch-tol 1e-2
run --kappa 10
run --n-coarse-max 2048
