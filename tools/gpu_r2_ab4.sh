#!/bin/bash
# same-box A/B: forward with x from L2 (3-stage ring, default) vs x through the TMA ring (GSPN_FWD_XTMA)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_build.log 2>&1 || { tail -30 gpurun_out/r2_build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -q -x -k "gpu_parity or pins or fullsize or merged or local or shards" > gpurun_out/r2_ab4_test.log 2>&1; tail -3 gpurun_out/r2_ab4_test.log
for c in 4 2; do
for i in 1 2 3; do
  for v in xg xtma; do
    if [ $v = xtma ]; then export GSPN_EXPERIMENTS=1 GSPN_FWD_XTMA=1; else unset GSPN_EXPERIMENTS GSPN_FWD_XTMA; fi
    python bench.py --config $c --steps 20 --warmup 5 --no-e2e --no-others --no-next --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); c=d['config']
print('cfg $c $v', 'value %.0f step %.4f fwd %.4f bwd %.4f clk %s %s' % (d['value'], d['ms_per_step'], c['fwd_ms'], c['bwd_ms'], d['clocks']['sm_mhz'], d['clocks']['reasons']))"
  done
done
done
