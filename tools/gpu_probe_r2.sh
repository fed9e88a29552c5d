#!/bin/bash
# round 2: TMA row-width probe + baseline bench at HEAD
set -x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tma_probe tools/tma_probe.cu
for cw in 16 32 64 128; do
  st=4; [ $cw = 128 ] && st=3
  /tmp/tma_probe $cw 148 2560 $st 0 1
done
/tmp/tma_probe 32 148 2560 6 0 1
/tmp/tma_probe 64 148 2560 6 0 1
/tmp/tma_probe 64 296 2560 3 0 1
/tmp/tma_probe 32 296 2560 3 0 1
python -c "import __graft_entry__ as g; g.build()"
python bench.py --steps 20 --warmup 5 > gpurun_out/r2_base_bench.log 2>&1
tail -3 gpurun_out/r2_base_bench.log
