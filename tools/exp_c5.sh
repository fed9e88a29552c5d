#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 600 ncu --metrics $M --clock-control none -k regex:"stream_kernel|out_" -s 3 -c 3 --csv \
    python bench.py --config 5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline 2>/dev/null | grep -E "stream_kernel|out_" > gpurun_out/exp_c5.csv
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fwd_stream" -s 1 -c 1 -o gpurun_out/prof_c5 -f \
  python bench.py --config 5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
