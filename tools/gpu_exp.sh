#!/bin/bash
export GSPN_EXPERIMENTS=1  # enable the library's experiment knobs (GSPN_*)
# tests + bench variants (bwd E) + ncu profile
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu --maxfail=10 -k "not config5" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for E in 2 4; do
  GSPN_BWD_E=$E timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_E$E.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bwd_stream_kernel -s 1 -c 1 -o gpurun_out/prof_bwd -f \
  python bench.py --config 4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/prof_bench.log 2>&1
