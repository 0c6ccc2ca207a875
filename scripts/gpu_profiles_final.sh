#!/bin/bash
# Profile pass for the committed summaries: launch list + full captures, collected on the box
mkdir -p gpurun_out/profiles_new
ROUND=r02 bash scripts/gpu_profile.sh
python scripts/profile_collect.py r02 > gpurun_out/profile_collect.log 2>&1
cp profiles/r02_ncu_full_summary.txt profiles/r02_launches* profiles/traffic.json gpurun_out/profiles_new/
ncu -i gpurun_out/r02_partition.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r02_partition_src.csv 2>/dev/null
ncu -i gpurun_out/r02_recompute.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r02_recompute_src.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
