#!/bin/bash
export GSPN_EXPERIMENTS=1  # enable the library's experiment knobs (GSPN_*)
# DRAM traffic of the fwd/bwd stream kernels per direction subset and L2 policy (ncu metrics pass)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
run() { # tag env dirs
  env $2 timeout 300 ncu --metrics $M --clock-control none -k regex:stream_kernel -s 2 -c 2 --csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --dirs $3 2>/dev/null | grep stream_kernel > gpurun_out/exp_$1.csv
}
run v_default "GSPN_POL=1,0,1,0,1,2" 0x3
run h_default "GSPN_POL=1,0,1,0,1,2" 0xC
run all_default "GSPN_POL=1,0,1,0,1,2" 0xF
run h_last "GSPN_POL=1,0,2,0,2,2" 0xC
run h_first "GSPN_POL=1,0,0,0,0,2" 0xC
run all_xlast "GSPN_POL=2,0,1,0,1,2" 0xF
run h_promo64 "GSPN_POL=1,0,1,0,1,2 GSPN_L2PROMO=64" 0xC
run h_promo256 "GSPN_POL=1,0,1,0,1,2 GSPN_L2PROMO=256" 0xC
run all_accnormal "GSPN_POL=1,0,1,0,1,1" 0xF
