#!/bin/bash
# one ncu --set full capture of kernels matching $NCU_K on bench config $NCU_CFG, summarised
mkdir -p gpurun_out
OUT=${NCU_OUT:-r2_ncu}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$NCU_K" -c ${NCU_C:-2} -o gpurun_out/$OUT -f \
  python bench.py --config ${NCU_CFG:-3b} --steps 1 --warmup 1 --no-e2e --no-others --no-next --no-cpu-baseline > gpurun_out/${OUT}.log 2>&1
echo "ncu rc=$?"
python tools/ncu_summary.py gpurun_out/$OUT.ncu-rep > gpurun_out/${OUT}.md 2>&1; echo "summary rc=$?"
head -80 gpurun_out/${OUT}.md
