#!/bin/bash
# ncu capture of the materialised select (knn_select) on short and headline-length rows.
mkdir -p gpurun_out
cap() {  # tag M N k
  timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k "regex:select" -s 1 -c 1 \
     -o gpurun_out/sel_$1 -f python scripts/select_bench.py $2,$3,$4 > gpurun_out/sel_$1.log 2>&1
  tail -1 gpurun_out/sel_$1.log
}
cap ${TAG:-}n4096 65536 4096 32
cap ${TAG:-}n65536 16384 65536 32
