#!/bin/bash
# ncu source capture of C4's large-k candidate select and quantile pivot kernels
mkdir -p gpurun_out
make -j16 > /dev/null 2>&1 || exit 1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"candidate_select_warp" -s 1 -c 1 \
  -o gpurun_out/c4 -f python bench.py --config C4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/c4.log 2>&1
ncu -i gpurun_out/c4.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/c4_src.csv 2>/dev/null
ncu -i gpurun_out/c4.ncu-rep --page details --csv > gpurun_out/c4_details.csv 2>/dev/null
rm -f gpurun_out/c4.ncu-rep
