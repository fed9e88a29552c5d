#!/bin/bash
export GSPN_EXPERIMENTS=1  # enable the library's experiment knobs (GSPN_*)
bash tools/gpu_check.sh
for PF in 0 1 2 3 4; do
  GSPN_PF=$PF timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 10 > gpurun_out/pf_$PF.log 2>&1
done
timeout 900 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5.log 2>&1
