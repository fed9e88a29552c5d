#!/bin/bash
mkdir -p gpurun_out
cd tools && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_probe tma_probe.cu && cd ..
M=gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct
for cw in 16 32 64 128; do
  for ctas in 74 148; do
    ./tools/tma_probe $cw $ctas 2560 4 0 1 >> gpurun_out/tma_probe.txt 2>&1
    ncu --metrics $M --clock-control none -k regex:probe -s 1 -c 1 --csv ./tools/tma_probe $cw $ctas 2560 4 0 1 2>/dev/null | grep probe | awk -F'","' '{print "'$cw' '$ctas'", $13, $15}' >> gpurun_out/tma_probe_ncu.txt
  done
done
for pol in 0 2; do
  ./tools/tma_probe 16 148 2560 4 0 $pol >> gpurun_out/tma_probe.txt 2>&1
  ncu --metrics $M --clock-control none -k regex:probe -s 1 -c 1 --csv ./tools/tma_probe 16 148 2560 4 0 $pol 2>/dev/null | grep probe | awk -F'","' '{print "16 148 pol'$pol'", $13, $15}' >> gpurun_out/tma_probe_ncu.txt
done
