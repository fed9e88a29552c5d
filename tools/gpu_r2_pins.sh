#!/bin/bash
# round 2: new parity pins (closed forms, force-split bitwise, fp32 3a/5, unrounded e2e), error log
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_build.log 2>&1 || { tail -30 gpurun_out/r2_build.log; exit 1; }
export GSPN_ERRLOG=gpurun_out/parity_errors.jsonl
rm -f $GSPN_ERRLOG
timeout 1800 python -m pytest tests -m gpu -q -x -k "pins or fullsize or end_to_end or fused_bwd or local_parity" > gpurun_out/r2_pins.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_pins.log
tail -30 gpurun_out/r2_pins.log
