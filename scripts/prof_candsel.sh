#!/bin/bash
# ncu source captures of the two candidate selects (headline k = 32, C4 k = 1024)
mkdir -p gpurun_out
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:candidate_select_kernel -s 1 -c 1 \
  -o gpurun_out/cs32 -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:candidate_select_warp -s 1 -c 1 \
  -o gpurun_out/cs1k -f python bench.py --config C4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
for r in cs32 cs1k; do
  ncu -i gpurun_out/$r.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${r}_src.csv 2>/dev/null
  ncu -i gpurun_out/$r.ncu-rep --page details --csv > gpurun_out/${r}_details.csv 2>/dev/null
done
rm -f gpurun_out/cs32.ncu-rep gpurun_out/cs1k.ncu-rep
