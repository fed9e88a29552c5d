#!/bin/bash
# round 2 iteration: build, targeted GPU tests, per-config bench lines, ncu of the changed kernels
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_build.log 2>&1 || { tail -30 gpurun_out/r2_build.log; exit 1; }
export GSPN_ERRLOG=gpurun_out/parity_errors_iter.jsonl
rm -f $GSPN_ERRLOG
timeout 1500 python -m pytest tests -m gpu -q -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/r2_iter_test.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_iter_test.log
tail -6 gpurun_out/r2_iter_test.log
for c in ${BENCH_CFGS:-3a 3b 4}; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-e2e --no-others --no-next --no-cpu-baseline > gpurun_out/r2_iter_bench_$c.log 2>&1
  python - "$c" <<'PY'
import json,sys
c=sys.argv[1]
l=[x for x in open(f"gpurun_out/r2_iter_bench_{c}.log") if x.startswith("{")]
if not l: print(c, "NO LINE"); print(open(f"gpurun_out/r2_iter_bench_{c}.log").read()[-2000:]); sys.exit()
d=json.loads(l[-1]); cf=d["config"]
print(c, "value %.0f GB/s step %.4f ms fwd %.4f bwd %.4f frac %.3f launches %s path %s" % (d["value"], d["ms_per_step"], cf["fwd_ms"], cf["bwd_ms"], d["roofline"]["frac"], d["launches_per_call"], cf["path"]))
PY
done
if [ -n "$NCU_K" ]; then
  ncu --set full --clock-control none --import-source on -k regex:$NCU_K -c ${NCU_C:-2} -o gpurun_out/r2_iter_prof -f python bench.py --config ${NCU_CFG:-3b} --steps 1 --warmup 1 --no-e2e --no-others --no-next --no-cpu-baseline > /dev/null 2>&1; echo ncu rc=$?
fi
