# session 5: streaming (evict-first) factor loads A/B at L=150/200; parity (default + L=48 production variants incl. ring); W=12 at M=130 with a 40k dense coarse block
mkdir -p gpurun_out
for v in "stream:" "nostream:AJ_LIB=paper_math_0508111_b200/libaj_nostream.so"; do
  name=${v%%:*}; envs=${v#*:}
  env $envs timeout 600 python scripts/prof_kernels.py 150 20 precond > gpurun_out/s5f_apply150_$name.log 2>&1; echo "$name: $(tail -1 gpurun_out/s5f_apply150_$name.log)"
  env $envs timeout 600 python scripts/prof_kernels.py 200 10 precond > gpurun_out/s5f_apply200_$name.log 2>&1; echo "L200 $name: $(tail -1 gpurun_out/s5f_apply200_$name.log)"
  env $envs timeout 300 python scripts/rep_solve.py 1 4 > gpurun_out/s5f_rep50_$name.jsonl 2>&1; tail -1 gpurun_out/s5f_rep50_$name.jsonl
done
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -k "precond" > gpurun_out/s5f_tests_precond.log 2>&1; echo "tests rc $?"; tail -3 gpurun_out/s5f_tests_precond.log
AJ_DENSE_CAP=40000 AJ_MAX_OUTER=300 AJ_VERBOSE=1 timeout 1500 python scripts/run_config.py 4 12 4 130 > gpurun_out/s5f_w12_L130.jsonl 2> gpurun_out/s5f_w12_L130.err; cut -c1-700 gpurun_out/s5f_w12_L130.jsonl; tail -3 gpurun_out/s5f_w12_L130.err | cut -c1-300
