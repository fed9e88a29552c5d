#!/bin/bash
# same-box A/B: single-launch backward with per-plane readiness (default) vs the grid-wide barrier
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_build.log 2>&1 || { tail -30 gpurun_out/r2_build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x -k "fused or merged or fullsize or pins or gpu_parity" > gpurun_out/r2_ab2_test.log 2>&1; tail -3 gpurun_out/r2_ab2_test.log
for i in 1 2 3; do
  for v in ready grid; do
    if [ $v = grid ]; then export GSPN_EXPERIMENTS=1 GSPN_GRID_BARRIER=1; else unset GSPN_EXPERIMENTS GSPN_GRID_BARRIER; fi
    python bench.py --config 4 --steps 20 --warmup 5 --no-e2e --no-others --no-next --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); c=d['config']
print('$v', 'value %.0f step %.4f fwd %.4f bwd %.4f clk %s %s' % (d['value'], d['ms_per_step'], c['fwd_ms'], c['bwd_ms'], d['clocks']['sm_mhz'], d['clocks']['reasons']))"
  done
done
