#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 12 --csv --log-file gpurun_out/launches_fused.csv \
  python bench.py --config 4 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-next > gpurun_out/launches_fused_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bwd_fused|bwd_dx" -s 2 -c 2 -o gpurun_out/prof_fused -f \
  python bench.py --config 4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-next > gpurun_out/prof_fused_bench.log 2>&1
