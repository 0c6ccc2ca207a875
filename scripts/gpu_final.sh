#!/bin/bash
# Round-end pass: full verification, config lines, reference arm, profiles.
mkdir -p gpurun_out
bash scripts/gpu_verify.sh
timeout -s KILL 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2>gpurun_out/bench_ref.err; cat gpurun_out/bench_ref.json
bash scripts/gpu_configs.sh > gpurun_out/configs.txt 2>&1; cat gpurun_out/configs.txt
KNN_PIVOT1=1 bash scripts/bench_brief.sh > gpurun_out/pivot1.txt 2>&1; cat gpurun_out/pivot1.txt
ROUND=r01 bash scripts/gpu_profile.sh
python scripts/profile_collect.py r01 > /dev/null 2>&1
mkdir -p gpurun_out/profiles_new; cp profiles/r01_ncu_full_summary.txt profiles/r01_launches* profiles/traffic.json gpurun_out/profiles_new/
ncu -i gpurun_out/r01_partition.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r01_partition_src.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
