# config 5 experiment A/B: cluster CTA size / stage count knobs
for rep in 1 2; do for v in "" "GSPN_CL_NWC=6 GSPN_NSTAGES=1" "GSPN_CL_NWC=5 GSPN_NSTAGES=1" "GSPN_CL_NWC=6"; do
  env GSPN_EXPERIMENTS=1 $v timeout 300 python bench.py --config 5 --steps 5 --warmup 2 --no-e2e --no-others --no-next --no-cpu-baseline 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['config']; print('[$v]', 'step %.4f fwd %.4f bwd %.4f' % (d['ms_per_step'], c['fwd_ms'], c['bwd_ms']))"
done; done
