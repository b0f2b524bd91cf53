#!/bin/bash
# JD time-to-5-eigenpairs over lattice sizes (configs W=16.5); one JSON line per size
for c in 2; do python scripts/run_config.py $c 2>>gpurun_out/jd_sizes.err | tee -a gpurun_out/jd_sizes.log; done
