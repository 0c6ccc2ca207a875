#!/bin/bash
# ncu source capture of the headline's single-product partition (dist_tc_kernel<0,1,5,SymSched>)
mkdir -p gpurun_out
make -j16 > /dev/null 2>&1 || exit 1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"\(int\)5, knn::tc::SymSched" -s 1 -c 1 \
  -o gpurun_out/p1 -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/p1.log 2>&1
ncu -i gpurun_out/p1.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/p1_src.csv 2>/dev/null
ncu -i gpurun_out/p1.ncu-rep --page details --csv > gpurun_out/p1_details.csv 2>/dev/null
ncu -i gpurun_out/p1.ncu-rep --page raw --csv > gpurun_out/p1_raw.csv 2>/dev/null
rm -f gpurun_out/p1.ncu-rep
