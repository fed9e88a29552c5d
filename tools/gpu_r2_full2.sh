#!/bin/bash
# round 2: full GPU suite with the error log, smoke, default bench line, ncu of config 5's forward
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_build.log 2>&1 || { tail -30 gpurun_out/r2_build.log; exit 1; }
export GSPN_ERRLOG=gpurun_out/parity_errors_full.jsonl
rm -f $GSPN_ERRLOG
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2_full_test.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_full_test.log
tail -4 gpurun_out/r2_full_test.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/r2_bench_default.log 2>&1; echo "bench rc=$?"
grep '^{' gpurun_out/r2_bench_default.log | tail -1 > gpurun_out/r2_bench_default.json
ncu --set full --clock-control none -k regex:"fwd_stream_kernel" -s 1 -c 1 -o gpurun_out/r2_cfg5_fwd_prof -f python bench.py --config 5 --steps 1 --warmup 1 --no-e2e --no-others --no-next --no-cpu-baseline > /dev/null 2>&1; echo "ncu cfg5 rc=$?"
du -sh gpurun_out
