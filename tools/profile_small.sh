#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_next.py -q -m gpu -k "small or local" > gpurun_out/pytest_small.log 2>&1
for c in 3a 3b; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-next > gpurun_out/bench_c$c.log 2>&1; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"small_kernel" -s 2 -c 2 -o gpurun_out/prof_small -f \
  python bench.py --config 3b --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-next > gpurun_out/prof_small_bench.log 2>&1
