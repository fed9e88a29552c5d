#!/bin/bash
# round 2: grouped small-plane kernels (configs 3a/3b) + shard tests + quick per-config bench
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_build.log 2>&1 || { tail -30 gpurun_out/r2_build.log; exit 1; }
export GSPN_ERRLOG=gpurun_out/parity_errors_small.jsonl
rm -f $GSPN_ERRLOG
timeout 1200 python -m pytest tests -m gpu -q -k "small or shards or 3a or 3b or local or smoke or parity" > gpurun_out/r2_small_test.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_small_test.log
tail -8 gpurun_out/r2_small_test.log
for c in 3a 3b; do timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-e2e --no-others --no-next --cpu-seconds 2 > gpurun_out/r2_bench_$c.log 2>&1; tail -c 1500 gpurun_out/r2_bench_$c.log; echo; done
ncu --set full --clock-control none -k regex:grp_small -c 2 -o gpurun_out/r2_small_prof -f python bench.py --config 3b --steps 1 --warmup 1 --no-e2e --no-others --no-next --no-cpu-baseline > /dev/null 2>&1; echo ncu rc=$?
