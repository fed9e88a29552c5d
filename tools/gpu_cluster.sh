#!/bin/bash
bash tools/gpu_check.sh
timeout 900 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c5.log
timeout 1200 python -m pytest tests -q -m gpu -k config5 > gpurun_out/pytest_c5.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_c5.log
