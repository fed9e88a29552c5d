#!/bin/bash
export GSPN_EXPERIMENTS=1  # enable the library's experiment knobs (GSPN_*)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for p in 0 64 128 256; do
  GSPN_L2PROMO=$p timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/sweep_promo$p.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stream_kernel -s 2 -c 2 -o gpurun_out/prof_cfg4 -f \
  python bench.py --config 4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/prof_bench.log 2>&1
