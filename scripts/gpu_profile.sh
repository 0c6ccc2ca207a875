#!/bin/bash
# Profile pass (never a bench number): launch list of the bench command and one full
# ncu capture of each hot kernel of the default plan.  Reports land in gpurun_out/.
mkdir -p gpurun_out
make -j8 > /dev/null || exit 1
R=${ROUND:-r01}
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${R}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
# pivot plan kernels, in launch order per step: sample GEMM, sample select, pivot prep,
# partition GEMM, candidate select; capture one of each (skip the warm-up step)
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:dist_tc -s 2 -c 2 \
    -o gpurun_out/${R}_dist_tc -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${R}_dist_tc.log 2>&1
tail -1 gpurun_out/${R}_dist_tc.log
for K in select_warp candidate_select prep_kernel; do
  timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 \
      -o gpurun_out/${R}_$K -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${R}_$K.log 2>&1
  tail -1 gpurun_out/${R}_$K.log
done
