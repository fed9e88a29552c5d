#!/bin/bash
# A/B: current gspn_stream.cu vs tools/ab/$1 on the same box (config 4 bench, 2 runs each)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for i in 1 2; do timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 10 > gpurun_out/ab_cur_$i.log 2>&1; done
cp paper_2512_07884_b200/csrc/gspn_stream.cu /tmp/cur.cu
cp tools/ab/$1 paper_2512_07884_b200/csrc/gspn_stream.cu
python -m paper_2512_07884_b200.build --force > gpurun_out/build_b.log 2>&1
for i in 1 2; do timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 10 > gpurun_out/ab_old_$i.log 2>&1; done
cp /tmp/cur.cu paper_2512_07884_b200/csrc/gspn_stream.cu
