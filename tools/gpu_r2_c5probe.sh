#!/bin/bash
# launch lists (per-kernel device times) of configs 5 and 3b, and config 5 bench line
mkdir -p gpurun_out
for c in 5 3b 3a; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r2_launches_cfg$c.csv \
    python bench.py --config $c --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-others --no-next > gpurun_out/r2_launches_cfg$c.log 2>&1
  echo "cfg $c ncu rc=$?"
done
timeout 300 python bench.py --config 5 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-others --no-next > gpurun_out/r2_c5_bench.log 2>&1; echo "bench rc=$?"
grep '^{' gpurun_out/r2_c5_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['config']; print('c5', d['value'], c['fwd_ms'], c['bwd_ms'], d['launches_per_call'])"
