#!/bin/bash
mkdir -p gpurun_out
make -j8 > /dev/null || exit 1
timeout -s KILL 300 python scripts/select_bench.py
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:select -s 1 -c 1 -o gpurun_out/prof_sel2 -f python scripts/select_bench.py > gpurun_out/ncu_sel2.log 2>&1; tail -2 gpurun_out/ncu_sel2.log
