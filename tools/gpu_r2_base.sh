#!/bin/bash
# round 2 baseline at HEAD: build, GPU suite, default bench, TMA row-width probe
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_gputest.log
tail -3 gpurun_out/r2_gputest.log
python bench.py --steps 20 --warmup 5 > gpurun_out/r2_base_bench.log 2>&1
tail -2 gpurun_out/r2_base_bench.log
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tma_probe tools/tma_probe.cu
for cw in 16 32 64 128; do
  st=4; [ $cw = 128 ] && st=3
  /tmp/tma_probe $cw 148 2560 $st 0 1
done > gpurun_out/r2_tma_probe.log 2>&1
/tmp/tma_probe 64 148 2560 6 0 1 >> gpurun_out/r2_tma_probe.log 2>&1
/tmp/tma_probe 64 296 2560 3 0 1 >> gpurun_out/r2_tma_probe.log 2>&1
cat gpurun_out/r2_tma_probe.log
