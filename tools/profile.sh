#!/bin/bash
# ncu launch list + full capture of the fwd and bwd stream kernels on the bench workload
mkdir -p gpurun_out
CFG=${CFG:-4}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_cfg${CFG}.csv \
  python bench.py --config $CFG --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/launches_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"stream_kernel|out_|fused" -s 3 -c 3 -o gpurun_out/prof_cfg${CFG} -f \
  python bench.py --config $CFG --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/prof_bench.log 2>&1
ls -la gpurun_out
