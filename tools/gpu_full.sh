#!/bin/bash
# build + smoke + gpu tests + bench + ncu profile of the bench workload
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -q -m gpu --maxfail=30 ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
if [ -n "$PROFILE" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stream_kernel -s 2 -c 2 -o gpurun_out/prof_cfg4 -f \
  python bench.py --config 4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/prof_bench.log 2>&1
fi
