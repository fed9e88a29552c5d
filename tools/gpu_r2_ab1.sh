#!/bin/bash
# same-box A/B: single-launch backward (default) vs the two-launch hybrid (GSPN_TWO_LAUNCH)
for i in 1 2 3; do
  for v in one two; do
    if [ $v = two ]; then export GSPN_EXPERIMENTS=1 GSPN_TWO_LAUNCH=1; else unset GSPN_EXPERIMENTS GSPN_TWO_LAUNCH; fi
    python bench.py --config 4 --steps 20 --warmup 5 --no-e2e --no-others --no-next --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); c=d['config']
print('$v', 'value %.0f step %.4f fwd %.4f bwd %.4f launches %s clk %s' % (d['value'], d['ms_per_step'], c['fwd_ms'], c['bwd_ms'], d['launches_per_call'], d['clocks']['sm_mhz']))"
  done
done
