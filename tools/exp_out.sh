#!/bin/bash
export GSPN_EXPERIMENTS=1  # enable the library's experiment knobs (GSPN_*)
# bwd output-kernel variants (GSPN_OUTK) + tests + bench + profile
bash tools/gpu_check.sh
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for K in 1 2 4; do
  GSPN_OUTK=$K timeout 300 ncu --metrics $M --clock-control none -k regex:"stream_kernel|out_" -s 3 -c 3 --csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline 2>/dev/null | grep -E "stream_kernel|out_" > gpurun_out/exp_outk$K.csv
done
bash tools/profile.sh
