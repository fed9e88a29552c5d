for rep in 1 2; do for v in "" "GSPN_OUT_RB=2" "GSPN_OUT_RB=8" "GSPN_OUT_RB=16"; do
  env GSPN_EXPERIMENTS=1 $v timeout 300 python bench.py --config 4 --steps 10 --warmup 3 --no-e2e --no-others --no-next --no-cpu-baseline 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['config']; print('c4 [$v]', 'step %.4f fwd %.4f bwd %.4f' % (d['ms_per_step'], c['fwd_ms'], c['bwd_ms']))"
done; done
for rep in 1 2; do for v in "" "GSPN_OUT_RB=56" "GSPN_OUT_RB=19" "GSPN_OUT_RB=14"; do
  env GSPN_EXPERIMENTS=1 $v timeout 300 python bench.py --config 2 --steps 20 --warmup 5 --no-e2e --no-others --no-next --no-cpu-baseline 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['config']; print('c2 [$v]', 'step %.4f fwd %.4f bwd %.4f' % (d['ms_per_step'], c['fwd_ms'], c['bwd_ms']))"
done; done
