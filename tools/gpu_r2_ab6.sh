#!/bin/bash
# same-box A/B: kHF backward (GSPN_HF, experiments) vs the default hybrid, configs 4 and 2
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_build.log 2>&1 || { tail -30 gpurun_out/r2_build.log; exit 1; }
timeout 300 python tools/hf_cmp.py 1,8,8,16,16,15,f32 1,2,2,300,264,15,bf16 2,2,2,512,512,15,bf16 1,3,3,200,136,15,bf16
for c in 4 2; do
for i in 1 2; do
  for v in hf hybrid; do
    unset GSPN_EXPERIMENTS GSPN_HF
    if [ $v = hf ]; then export GSPN_EXPERIMENTS=1 GSPN_HF=1; fi
    python bench.py --config $c --steps 20 --warmup 5 --no-e2e --no-others --no-next --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); c=d['config']
print('cfg $c $v', 'value %.0f step %.4f fwd %.4f bwd %.4f clk %s %s' % (d['value'], d['ms_per_step'], c['fwd_ms'], c['bwd_ms'], d['clocks']['sm_mhz'], d['clocks']['reasons']))"
  done
done
done
