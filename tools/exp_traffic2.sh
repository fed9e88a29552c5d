#!/bin/bash
export GSPN_EXPERIMENTS=1  # enable the library's experiment knobs (GSPN_*)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
run() { # tag env dirs
  env $2 timeout 300 ncu --metrics $M --clock-control none -k regex:stream_kernel -s 2 -c 2 --csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --dirs $3 2>/dev/null | grep stream_kernel > gpurun_out/exp2_$1.csv
}
run v "GSPN_X=1" 0x3
run h "GSPN_X=1" 0xC
run all_hstore_last "GSPN_POL=1,0,1,0,2,2" 0xF
run all_acc_normal "GSPN_POL=1,0,1,0,1,1" 0xF
run all_acc_first "GSPN_POL=1,0,1,0,1,0" 0xF
run all_x_first "GSPN_POL=0,0,1,0,1,2" 0xF
run all_hin_last "GSPN_POL=1,0,2,0,1,2" 0xF
run all_hin_first "GSPN_POL=1,0,0,0,1,2" 0xF
