# session 4: apply prefetch depth (PREF 8 / 12 / 16 entries per lane) at L=150; fp32-stored factor with the paper's drop rule
mkdir -p gpurun_out
for v in "default:" "p16l16:AJ_LIB=paper_math_0508111_b200/libaj_pref16.so AJ_PER_LANE=16" "p16l8:AJ_LIB=paper_math_0508111_b200/libaj_pref16.so" "p12l12:AJ_LIB=paper_math_0508111_b200/libaj_pref12.so AJ_PER_LANE=12"; do
  name=${v%%:*}; envs=${v#*:}
  env $envs timeout 600 python scripts/prof_kernels.py 150 20 precond > gpurun_out/s4d_apply150_$name.log 2>&1; echo "$name: $(tail -2 gpurun_out/s4d_apply150_$name.log | tr '\n' ' ')"
done
AJ_F32=1 timeout 600 python scripts/run_config.py 2 > gpurun_out/s4d_f32_L100.jsonl 2> gpurun_out/s4d_f32_L100.err; cut -c1-400 gpurun_out/s4d_f32_L100.jsonl
timeout 600 python scripts/run_config.py 2 > gpurun_out/s4d_f64_L100.jsonl 2> gpurun_out/s4d_f64_L100.err; cut -c1-400 gpurun_out/s4d_f64_L100.jsonl
