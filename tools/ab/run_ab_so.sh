#!/bin/bash
# A/B of two prebuilt libgspn.so on one box: current build vs tools/ab/libgspn_prev.so (config 4 bench, global
# scan only, alternating runs)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
cp paper_2512_07884_b200/lib/libgspn.so /tmp/libgspn_cur.so
for i in 1 2 3; do
  cp /tmp/libgspn_cur.so paper_2512_07884_b200/lib/libgspn.so
  timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-next --steps 10 > gpurun_out/ab_cur_$i.log 2>&1
  cp tools/ab/libgspn_prev.so paper_2512_07884_b200/lib/libgspn.so
  timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-next --steps 10 > gpurun_out/ab_prev_$i.log 2>&1
done
cp /tmp/libgspn_cur.so paper_2512_07884_b200/lib/libgspn.so
