#!/bin/bash
# same-box A/B of the in-tree library against builds under build_ab/ (GSPN_LIB, experiments only):
#   CFGS="2 4" LIBS="build_ab/libgspn_X.so" bash tools/ab_lib.sh
for c in ${CFGS:-2}; do
  for rep in 1 2; do
    for lib in default ${LIBS}; do
      if [ "$lib" = default ]; then unset GSPN_EXPERIMENTS GSPN_LIB; else export GSPN_EXPERIMENTS=1 GSPN_LIB=$lib; fi
      timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-e2e --no-others --no-next --no-cpu-baseline 2>/dev/null | grep '^{' | \
        python -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['config']; print('cfg $c rep $rep $lib', 'step %.4f fwd %.4f bwd %.4f' % (d['ms_per_step'], c['fwd_ms'], c['bwd_ms']))"
    done
  done
done
