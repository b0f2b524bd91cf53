# session 5: coarse cutover at L=50 (configs[1]); seeds of the JD start vector to separate the apply effect from the JD path
mkdir -p gpurun_out
for nc in 1024 1536 2048 3072 4096; do
  AJ_NCOARSE=$nc timeout 300 python scripts/rep_solve.py 1 4 > gpurun_out/s5h_rep50_nc$nc.jsonl 2>&1; echo "nc=$nc: $(tail -1 gpurun_out/s5h_rep50_nc$nc.jsonl)"
done
for nc in 1024 2048 4096; do
  AJ_NCOARSE=$nc timeout 300 python scripts/rep_solve.py 2 3 > gpurun_out/s5h_rep100_nc$nc.jsonl 2>&1; echo "L100 nc=$nc: $(tail -1 gpurun_out/s5h_rep100_nc$nc.jsonl)"
done
