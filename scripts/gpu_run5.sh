# DRAM traffic per preconditioner apply (ncu, per-kernel dram bytes) at L=50 (bench workload) and L=150
mkdir -p gpurun_out
for L in 50 150; do
  seed=1; [ $L = 150 ] && seed=4
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_apply|k_dense_mv|k_gj" --csv --log-file gpurun_out/traffic$L.csv python scripts/prof_kernels.py $L 1 precond $seed > gpurun_out/traffic$L.log 2>&1; echo "L=$L rc=$?"
done
