#!/bin/bash
# round 2: default bench line, launch list, one ncu --set full capture of the single-launch backward
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_build.log 2>&1 || { tail -30 gpurun_out/r2_build.log; exit 1; }
timeout 900 python bench.py > gpurun_out/r2_bench_default.log 2>&1; echo "bench rc=$?"
grep '^{' gpurun_out/r2_bench_default.log | tail -1 > gpurun_out/r2_bench_default.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/r2_cfg4_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-others --no-next --no-cpu-baseline > /dev/null 2>&1; echo "ncu launches rc=$?"
ncu --set full --clock-control none -k regex:"${NCU_K:-bwd_one}" -s ${NCU_S:-1} -c 1 -o gpurun_out/r2_${NCU_TAG:-cfg4_bwd}_prof -f python bench.py --config ${NCU_CFG:-4} --steps 1 --warmup 1 --no-e2e --no-others --no-next --no-cpu-baseline > /dev/null 2>&1; echo "ncu full rc=$?"
ls -la gpurun_out/
