#!/bin/bash
# DRAM traffic of the partition GEMM with parts of its epilogue disabled (KNN_DBG_EPI;
# wrong results, diagnostic only): where do the reads beyond the operands come from?
mkdir -p gpurun_out
for dbg in ${DBGS:-0 8 2 4}; do
  KNN_DBG_EPI=$dbg timeout -s KILL 600 ncu --clock-control none --kernel-name-base demangled -k regex:SymSched -s ${SKIP:-2} -c 1 \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_write.sum,lts__t_sectors_op_read.sum,lts__t_sectors_op_atom.sum \
    --csv python scripts/epi_cost.py > gpurun_out/ptraffic_$dbg.csv 2>&1
  echo "== dbg $dbg"; grep -E "dram__|gpu__time|lts__" gpurun_out/ptraffic_$dbg.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done
