#!/bin/bash
# One GPU session: bench + launch list + ncu captures of the top kernels.
set -x
mkdir -p gpurun_out
make -j8 > /dev/null
timeout -s KILL 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
cat gpurun_out/bench.json
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
tail -5 gpurun_out/launches.csv
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:dist_tc -s 1 -c 1 \
    -o gpurun_out/prof_gemm -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_gemm.log 2>&1
tail -3 gpurun_out/ncu_gemm.log
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:select_rows -s 1 -c 1 \
    -o gpurun_out/prof_select -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_select.log 2>&1
tail -3 gpurun_out/ncu_select.log
