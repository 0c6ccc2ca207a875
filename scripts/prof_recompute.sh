#!/bin/bash
# ncu source capture of the re-evaluation kernel (headline), and the pivot / decide kernels
mkdir -p gpurun_out
make -j16 > /dev/null 2>&1 || exit 1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"candidate_recompute|pivot_from_mins|pivot1_decide" -s 3 -c 3 \
  -o gpurun_out/rc -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/rc.log 2>&1
ncu -i gpurun_out/rc.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/rc_src.csv 2>/dev/null
ncu -i gpurun_out/rc.ncu-rep --page details --csv > gpurun_out/rc_details.csv 2>/dev/null
rm -f gpurun_out/rc.ncu-rep
