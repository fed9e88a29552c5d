#!/bin/bash
# round 2 final (session 3): GPU suite + error log, smoke, default bench line, launch list, ncu captures
mkdir -p gpurun_out
export GSPN_ERRLOG=gpurun_out/parity_errors_final.jsonl
rm -f $GSPN_ERRLOG
if [ -z "$SKIP_TESTS" ]; then timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2f_test.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2f_test.log; fi
tail -3 gpurun_out/r2f_test.log
unset GSPN_ERRLOG
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2f_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/r2f_bench.log 2>&1; echo "bench rc=$?"
grep '^{' gpurun_out/r2f_bench.log | tail -1 > gpurun_out/r2f_bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/r2f_launches_cfg4.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-next --no-others > /dev/null 2>&1; echo "ncu list rc=$?"
for c in 5 3a 3b 2; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/r2f_launches_cfg$c.csv \
    python bench.py --config $c --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-next --no-others > /dev/null 2>&1; echo "ncu list $c rc=$?"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bwd_one|fwd_stream" -s 2 -c 2 -o gpurun_out/r2f_cfg4 -f \
  python bench.py --config 4 --steps 1 --warmup 1 --no-e2e --no-others --no-next --no-cpu-baseline > /dev/null 2>&1; echo "ncu cfg4 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"stream_kernel|out_grp" -c 3 -o gpurun_out/r2f_cfg5 -f \
  python bench.py --config 5 --steps 1 --warmup 1 --no-e2e --no-others --no-next --no-cpu-baseline > /dev/null 2>&1; echo "ncu cfg5 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"grp" -c 2 -o gpurun_out/r2f_cfg3a -f \
  python bench.py --config 3a --steps 1 --warmup 1 --no-e2e --no-others --no-next --no-cpu-baseline > /dev/null 2>&1; echo "ncu cfg3a rc=$?"
for r in r2f_cfg4 r2f_cfg5 r2f_cfg3a; do
  python tools/ncu_summary.py gpurun_out/$r.ncu-rep > gpurun_out/$r.md 2>&1
  ncu -i gpurun_out/$r.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/$r.src.csv 2>/dev/null
  python tools/ncu_lines.py gpurun_out/$r.src.csv 40 > gpurun_out/$r.lines.txt 2>&1
  rm -f gpurun_out/$r.ncu-rep gpurun_out/$r.src.csv   # gpurun copies back <= 64 MiB
done
ls -la gpurun_out | tail -20
