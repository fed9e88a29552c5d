#!/bin/bash
# round 2 (session 3): full GPU suite with the error log, smoke, default bench line, launch list of the default bench
mkdir -p gpurun_out
export GSPN_ERRLOG=gpurun_out/parity_errors_full3.jsonl
rm -f $GSPN_ERRLOG
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2_full3_test.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_full3_test.log
tail -4 gpurun_out/r2_full3_test.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_full3_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/r2_full3_bench.log 2>&1; echo "bench rc=$?"
grep '^{' gpurun_out/r2_full3_bench.log | tail -1 > gpurun_out/r2_full3_bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/r2_full3_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-next --no-others > /dev/null 2>&1; echo "ncu rc=$?"
