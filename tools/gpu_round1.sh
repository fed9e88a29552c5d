#!/bin/bash
# first GPU round: build, smoke, gpu tests, short bench
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1200 python -m pytest tests -x -q -m gpu -k "not config5" > gpurun_out/pytest_gpu.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e > gpurun_out/bench.log 2>&1
