#!/bin/bash
# round 2: full GPU suite with the normwise error log, then the default bench line
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_build.log 2>&1 || { tail -30 gpurun_out/r2_build.log; exit 1; }
export GSPN_ERRLOG=gpurun_out/parity_errors.jsonl
rm -f $GSPN_ERRLOG
timeout 2400 python -m pytest tests -m gpu -q ${PYTEST_ARGS:-} > gpurun_out/r2_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_gputest.log
tail -15 gpurun_out/r2_gputest.log
timeout 900 python bench.py ${BENCH_ARGS:---steps 20 --warmup 5} > gpurun_out/r2_bench.log 2>&1; echo "bench rc=$?"
tail -c 6000 gpurun_out/r2_bench.log
