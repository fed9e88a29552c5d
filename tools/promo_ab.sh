for rep in 1 2; do for v in 0 64 128 256; do
  GSPN_EXPERIMENTS=1 GSPN_L2PROMO=$v timeout 300 python bench.py --config 4 --steps 10 --warmup 3 --no-e2e --no-others --no-next --no-cpu-baseline 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['config']; print('promo $v', 'step %.4f fwd %.4f bwd %.4f' % (d['ms_per_step'], c['fwd_ms'], c['bwd_ms']))"
done; done
