#!/bin/bash
# Round measurements: default bench line (and the 3-product plan), configs, profile pass
mkdir -p gpurun_out
make -j16 > /dev/null || exit 1
timeout -s KILL 600 python bench.py > gpurun_out/bench_r02.json 2> gpurun_out/bench_r02.err; tail -2 gpurun_out/bench_r02.err
python3 scripts/bench_summary.py gpurun_out/bench_r02.json
KNN_PIVOT1=0 timeout -s KILL 600 python bench.py --no-cpu-baseline > gpurun_out/bench_r02_exact.json 2>/dev/null
python3 scripts/bench_summary.py gpurun_out/bench_r02_exact.json
ROUND=r02 bash scripts/gpu_profile.sh
python scripts/profile_collect.py r02 > /dev/null 2>&1
mkdir -p gpurun_out/profiles_new; cp profiles/r02_ncu_full_summary.txt profiles/r02_launches* profiles/traffic.json gpurun_out/profiles_new/
ncu -i gpurun_out/r02_partition.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r02_partition_src.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
