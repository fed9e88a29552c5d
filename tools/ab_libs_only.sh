#!/bin/bash
# same-box A/B of builds under build_ab/ only (GSPN_LIB, experiments only), interleaved reps:
#   CFGS="4" LIBS="build_ab/a.so build_ab/b.so" REPS=3 bash tools/ab_libs_only.sh
export GSPN_EXPERIMENTS=1
for c in ${CFGS:-4}; do
  for rep in $(seq ${REPS:-3}); do
    for lib in ${LIBS}; do
      GSPN_LIB=$lib timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-e2e --no-others --no-next --no-cpu-baseline 2>/dev/null | grep '^{' | \
        python -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['config']; print('cfg $c rep $rep $lib', 'step %.4f fwd %.4f bwd %.4f' % (d['ms_per_step'], c['fwd_ms'], c['bwd_ms']))"
    done
  done
done
