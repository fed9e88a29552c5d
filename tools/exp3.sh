#!/bin/bash
export GSPN_EXPERIMENTS=1  # enable the library's experiment knobs (GSPN_*)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
run() { # tag env dirs
  env $2 timeout 300 ncu --metrics $M --clock-control none -k regex:stream_kernel -s 2 -c 2 --csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --dirs $3 2>/dev/null | grep stream_kernel > gpurun_out/exp3_$1.csv
}
run all_default "X=1" 0xF
run all_null "GSPN_NULL=1" 0xF
run v_null "GSPN_NULL=1" 0x3
run h_null "GSPN_NULL=1" 0xC
run all_nosleep "GSPN_NOSLEEP=1" 0xF
run all_promo64 "GSPN_L2PROMO=64" 0xF
run all_promo128 "GSPN_L2PROMO=128" 0xF
run h_promo128 "GSPN_L2PROMO=128" 0xC
run all_fwd1 "GSPN_FWD_CTAS=1" 0xF
