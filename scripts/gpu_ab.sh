#!/bin/bash
# A/B of ablibs/old.so vs ablibs/new.so (alternating bench lines), then the epilogue
# diagnostic of new, then (optional, NCU=1) a full ncu capture of new's partition kernel.
mkdir -p gpurun_out
for i in 1 2 3; do
  for v in old new; do echo "== $v"; KNN_LIB_PATH=ablibs/$v.so bash scripts/bench_brief.sh --steps ${STEPS:-30} ${BENCH_ARGS} | head -${LINES_AB:-2}; done
done
if [ -n "$DIAG" ]; then
  for d in 0 4 2 16 8; do KNN_LIB_PATH=ablibs/new.so KNN_DBG_EPI=$d timeout 120 python scripts/epi_cost.py 2>&1 | tail -1; done
fi
if [ -n "$NCU" ]; then
  KNN_LIB_PATH=ablibs/new.so timeout -s KILL 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:SymSched" -s 1 -c 1 \
      -o gpurun_out/ab_partition -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ab_ncu.log 2>&1
  tail -2 gpurun_out/ab_ncu.log
fi
