#!/bin/bash
# Profile pass (never a bench number): launch list of the bench command and one full
# ncu capture of each hot kernel.  Reports land in gpurun_out/, summaries go to profiles/.
mkdir -p gpurun_out
make -j8 > /dev/null || exit 1
R=${ROUND:-r01}
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${R}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
for K in dist_tc select_warp prep; do
  timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 \
      -o gpurun_out/${R}_$K -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${R}_$K.log 2>&1
  tail -1 gpurun_out/${R}_$K.log
done
