mkdir -p gpurun_out
for c in "precond_apply,precond_setup" "spmv,precond_apply,precond_setup" "precond_apply,precond_setup"; do
python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-e2e --big-L 0 --precond-L 0 --prof-cats $c 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$c', round(d['value']*1e3,1), [round(x,1) for x in d['step_ms']])"
done
