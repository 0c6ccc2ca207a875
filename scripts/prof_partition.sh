#!/bin/bash
# ncu full capture (with source) of the headline's partition GEMM (pivot plan, SYM).
mkdir -p gpurun_out
make -j8 > /dev/null || exit 1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:SymSched -s 1 -c 1 \
  -o gpurun_out/partition -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/partition.log 2>&1
tail -2 gpurun_out/partition.log
