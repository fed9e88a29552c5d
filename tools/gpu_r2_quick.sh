#!/bin/bash
# quick A/B: bench lines of the given configs (default 5 4), then the GPU suite (optionally filtered)
mkdir -p gpurun_out
for c in ${BENCH_CFGS:-5 4}; do
  for v in ${VARIANTS:-default}; do
    if [ "$v" = default ]; then unset GSPN_EXPERIMENTS; else export GSPN_EXPERIMENTS=1; export $v=1; fi
    timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-others --no-next --no-cpu-baseline > gpurun_out/q_bench_${c}_$v.log 2>&1
    python - "$c" "$v" <<'PY'
import json,sys
c,v=sys.argv[1],sys.argv[2]
l=[x for x in open(f"gpurun_out/q_bench_{c}_{v}.log") if x.startswith("{")]
if not l: print(c, v, "NO LINE"); print(open(f"gpurun_out/q_bench_{c}_{v}.log").read()[-3000:]); sys.exit()
d=json.loads(l[-1]); cf=d["config"]
print(c, v, "value %.0f GB/s step %.4f ms fwd %.4f bwd %.4f frac %.3f launches %s path %s parity %s" % (d["value"], d["ms_per_step"], cf["fwd_ms"], cf["bwd_ms"], d["roofline"]["frac"], d["launches_per_call"], cf["path"], d.get("parity")))
PY
    if [ "$v" != default ]; then unset $v; fi
  done
done
unset GSPN_EXPERIMENTS
if [ -n "$RUN_TESTS" ]; then
  export GSPN_ERRLOG=gpurun_out/q_parity_errors.jsonl
  timeout ${TEST_TIMEOUT:-1500} python -m pytest tests -m gpu -q -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/q_test.log 2>&1; echo "pytest rc=$?" >> gpurun_out/q_test.log
  tail -5 gpurun_out/q_test.log
fi
