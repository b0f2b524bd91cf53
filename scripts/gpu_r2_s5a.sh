# session 5: coarse cutover size (n_coarse_max 1024 / 4096 / 8192) at L=150 and L=200; W=12 at the paper's largest W=12 size (M=130)
mkdir -p gpurun_out
for nc in 1024 4096 8192; do
  AJ_NCOARSE=$nc AJ_DENSE_CAP=16384 timeout 600 python scripts/run_config.py 3 16.5 3 150 > gpurun_out/s5a_L150_nc$nc.jsonl 2> gpurun_out/s5a_L150_nc$nc.err; cut -c1-330 gpurun_out/s5a_L150_nc$nc.jsonl
done
for nc in 4096 8192; do
  AJ_NCOARSE=$nc AJ_DENSE_CAP=16384 timeout 600 python scripts/run_config.py 3 > gpurun_out/s5a_L200_nc$nc.jsonl 2> gpurun_out/s5a_L200_nc$nc.err; cut -c1-330 gpurun_out/s5a_L200_nc$nc.jsonl
done
AJ_DENSE_CAP=24576 AJ_MAX_OUTER=300 timeout 1500 python scripts/run_config.py 4 12 4 130 > gpurun_out/s5a_w12_L130.jsonl 2> gpurun_out/s5a_w12_L130.err; cut -c1-600 gpurun_out/s5a_w12_L130.jsonl
