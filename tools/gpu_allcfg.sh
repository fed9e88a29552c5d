#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for c in 1 2 3a 3b 5; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 5 --warmup 3 > gpurun_out/bench_cfg$c.log 2>&1
done
