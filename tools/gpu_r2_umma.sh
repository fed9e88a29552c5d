#!/bin/bash
# round 2: tcgen05 proxy projections -- parity, timing vs SIMT, ncu capture
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_build.log 2>&1 || { tail -30 gpurun_out/r2_build.log; exit 1; }
export GSPN_ERRLOG=gpurun_out/parity_errors_umma.jsonl
rm -f $GSPN_ERRLOG
timeout 900 python -m pytest tests -m gpu -q -k "proxy" > gpurun_out/r2_umma_test.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_umma_test.log
tail -4 gpurun_out/r2_umma_test.log
cat > /tmp/proxy_run.py <<'PY'
import sys, torch, paper_2512_07884_b200 as gspn
B, C, Cp, H, W = 1, 320, 40, 2048, 2048
dev = torch.device("cuda:0"); g = torch.Generator(device=dev).manual_seed(1)
x = (torch.rand((B, C, H, W), generator=g, device=dev) * 2 - 1).to(torch.bfloat16)
P = ((torch.rand((Cp, C), generator=g, device=dev) * 2 - 1) / C ** 0.5).to(torch.bfloat16)
Q = ((torch.rand((C, Cp), generator=g, device=dev) * 2 - 1) / Cp ** 0.5).to(torch.bfloat16)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    xp = gspn.proxy_mix(x, P); y = gspn.proxy_mix(xp, Q); dP = gspn.proxy_wgrad(xp, x)
torch.cuda.synchronize()
PY
ncu --set full --clock-control none --import-source on -k regex:umma -s 3 -c 3 -o gpurun_out/r2_umma_prof -f python tools/proxy_run.py 3 > gpurun_out/r2_umma_ncu.log 2>&1; echo ncu rc=$?
python bench.py --config 4 --steps 5 --warmup 3 --no-e2e --no-others --no-cpu-baseline > gpurun_out/r2_umma_bench.log 2>&1
python - <<'PY'
import json
l=[x for x in open("gpurun_out/r2_umma_bench.log") if x.startswith("{")]
d=json.loads(l[-1]); print(json.dumps(d["next"]["proxy"], indent=1))
PY
