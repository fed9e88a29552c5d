#!/bin/bash
# build + GPU tests of the §8(f) rows + the full GPU suite + short bench
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_next.py -q -m gpu --maxfail=40 > gpurun_out/pytest_next.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_next.log
timeout 1200 python -m pytest tests -q -m gpu --maxfail=30 --deselect tests/test_gpu_next.py > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
