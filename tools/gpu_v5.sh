#!/bin/bash
export GSPN_EXPERIMENTS=1  # enable the library's experiment knobs (GSPN_*)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -q -m gpu --maxfail=10 -k "not config5" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
run() { # tag env dirs
  env $2 timeout 300 ncu --metrics $M --clock-control none -k regex:"stream_kernel|dw_kernel" -s 3 -c 3 --csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --dirs $3 2>/dev/null | grep -E "stream_kernel|dw_kernel" > gpurun_out/exp5_$1.csv
}
run all "X=1" 0xF
run all_null "GSPN_NULL=1" 0xF
run v "X=1" 0x3
run h "X=1" 0xC
run all_E4 "GSPN_E=4" 0xF
