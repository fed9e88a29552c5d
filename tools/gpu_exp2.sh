#!/bin/bash
export GSPN_EXPERIMENTS=1  # enable the library's experiment knobs (GSPN_*)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -q -m gpu --maxfail=10 -k "not config5" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for v in "GSPN_FWD_CTAS=2" "GSPN_FWD_CTAS=1" "GSPN_FWD_CTAS=1 GSPN_PAIR=0"; do
  tag=$(echo $v | tr ' =' '__')
  env $v timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_$tag.log 2>&1
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 300 ncu --metrics $M --clock-control none -k regex:stream_kernel -s 2 -c 2 --csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline 2>/dev/null | grep stream_kernel > gpurun_out/exp_v4_default.csv
GSPN_FWD_CTAS=1 timeout 300 ncu --metrics $M --clock-control none -k regex:stream_kernel -s 2 -c 2 --csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline 2>/dev/null | grep stream_kernel > gpurun_out/exp_v4_fwd1.csv
