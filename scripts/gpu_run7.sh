mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "sqmr or precond_parity or jd_config0 or host or graph" > gpurun_out/pt.log 2>&1; tail -2 gpurun_out/pt.log
for i in 1 2 3; do
python bench.py --steps 12 --warmup 3 --no-cpu-baseline --no-e2e --big-L 0 --precond-L 0 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value']*1e3,1), [round(x) for x in d['step_ms']])"
done
