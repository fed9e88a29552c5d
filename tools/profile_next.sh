#!/bin/bash
# ncu --set full of the SURVEY §8(f) kernels (merge, GSPN-local, proxy) on the bench's next rows, and of the
# small-plane path on config 3b
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"merge_|mix_|wgrad_kernel" -c 8 -o gpurun_out/prof_next -f \
  python bench.py --config 4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/prof_next.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"small_kernel" -s 2 -c 2 -o gpurun_out/prof_small -f \
  python bench.py --config 3b --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-next > gpurun_out/prof_small.log 2>&1
