#!/bin/bash
export GSPN_EXPERIMENTS=1  # enable the library's experiment knobs (GSPN_*)
bash tools/gpu_check.sh
timeout 600 python bench.py --config 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_c2.log 2>&1
GSPN_NOPACK=1 timeout 600 python bench.py --config 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_c2_nopack.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 300 ncu --metrics $M --clock-control none -k regex:"stream_kernel|out_" -s 3 -c 3 --csv \
    python bench.py --config 2 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline 2>/dev/null | grep -E "stream_kernel|out_" > gpurun_out/exp_c2.csv
