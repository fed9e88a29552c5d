#!/bin/bash
export GSPN_EXPERIMENTS=1  # enable the library's experiment knobs (GSPN_*)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct
run() { # tag env dirs
  env $2 timeout 300 ncu --metrics $M --clock-control none -k regex:stream_kernel -s 2 -c 2 --csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --dirs $3 2>/dev/null | grep stream_kernel > gpurun_out/exp_$1.csv
}
for g in 16 37 74 148 296; do run h_grid$g "GSPN_GRID=$g" 0xC; done
for g in 37 74; do run v_grid$g "GSPN_GRID=$g" 0x3; done
