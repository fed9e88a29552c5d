for rep in 1 2; do for v in "" "GSPN_OUT_RBMAX=32" "GSPN_OUT_RBMAX=32 GSPN_OUT_RBBAL=1" "GSPN_OUT_RBBAL=1" "GSPN_OUT_RBMAX=64 GSPN_OUT_RBBAL=1"; do
  env GSPN_EXPERIMENTS=1 $v timeout 300 python bench.py --config ${CFG:-2} --steps 20 --warmup 5 --no-e2e --no-others --no-next --no-cpu-baseline 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['config']; print('[$v]', 'step %.4f fwd %.4f bwd %.4f' % (d['ms_per_step'], c['fwd_ms'], c['bwd_ms']))"
done; done
