#!/bin/bash
mkdir -p gpurun_out
M=gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 ncu --metrics $M --clock-control none -k regex:"stream_kernel" -s 2 -c 2 --csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline 2>/dev/null | grep -E "stream_kernel" > gpurun_out/ab_ncu_cur.csv
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fwd_stream" -s 1 -c 1 -o gpurun_out/ab_cur -f \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
cp paper_2512_07884_b200/csrc/gspn_stream.cu /tmp/cur.cu
cp tools/ab/$1 paper_2512_07884_b200/csrc/gspn_stream.cu
python -m paper_2512_07884_b200.build --force > gpurun_out/build_b.log 2>&1
timeout 300 ncu --metrics $M --clock-control none -k regex:"stream_kernel" -s 2 -c 2 --csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline 2>/dev/null | grep -E "stream_kernel" > gpurun_out/ab_ncu_old.csv
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fwd_stream" -s 1 -c 1 -o gpurun_out/ab_old -f \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
cp /tmp/cur.cu paper_2512_07884_b200/csrc/gspn_stream.cu
