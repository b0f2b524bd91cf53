mkdir -p gpurun_out
for ms in 200 500 1000 200 500 1000; do
AJ_CLOCK_MS=$ms python bench.py --steps 12 --warmup 3 --no-cpu-baseline --no-e2e --big-L 0 --precond-L 0 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$ms', round(d['value']*1e3,1), round(max(d['step_ms']),1), d['clocks']['samples'])"
done
