# tau_virtual trade-off at L=50 / 100 / 150 (setup vs JD iterations)
mkdir -p gpurun_out
for f in 10 20; do
  tv50=$(python -c "print($f*0.002)"); tv100=$(python -c "print($f*0.0005)"); tv150=$(python -c "print($f*2e-3*(50/150)**2)")
  AJ_TV=$tv50 timeout 400 python scripts/run_config.py 1 > gpurun_out/tv50_$f.log 2>&1; echo "L50 tv=${f}td"; tail -1 gpurun_out/tv50_$f.log | cut -c1-250
  AJ_TV=$tv100 AJ_MAX_OUTER=200 timeout 400 python scripts/run_config.py 2 > gpurun_out/tv100_$f.log 2>&1; echo "L100 tv=${f}td"; tail -1 gpurun_out/tv100_$f.log | cut -c1-250
  AJ_TV=$tv150 AJ_MAX_OUTER=200 timeout 600 python scripts/run_config.py 2 16.5 2 150 > gpurun_out/tv150_$f.log 2>&1; echo "L150 tv=${f}td"; tail -1 gpurun_out/tv150_$f.log | cut -c1-250
done
