#!/bin/bash
# Profile pass (never a bench number): launch list of the bench command and one full
# ncu capture of each kernel of the default plan (headline: the single-product pivot plan
# chosen on the device) and of the 3-product partition (KNN_PIVOT1=0).  Reports land in
# gpurun_out/; scripts/profile_collect.py turns them into profiles/ summaries.
mkdir -p gpurun_out
make -j8 > /dev/null || exit 1
R=${ROUND:-r02}
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${R}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
# one launch of each kernel of the step (skip the warm-up step's)
cap() {  # name regex
  timeout -s KILL 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k "regex:$2" -s 1 -c 1 -o gpurun_out/${R}_$1 -f $B > gpurun_out/${R}_$1.log 2>&1
  tail -1 gpurun_out/${R}_$1.log
}
cap partition "\(int\)5, knn::tc::SymSched"
cap recompute "candidate_recompute"
cap sample "\(int\)2, knn::tc::PanelSched"
cap pivot "pivot_from_mins"
cap prep "prep_kernel"
KNN_PIVOT1=0 cap partition3 "\(int\)1, knn::tc::SymSched"
KNN_PIVOT1=0 cap candsel "candidate_select_kernel"
# C4 (k = 1024): the quantile-pivot plan's own kernels
B="python bench.py --config C4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
cap c4_candsel "candidate_select_warp"
cap c4_pivot "pivot_from_sample"
cap c4_sample "\(int\)3, knn::tc::TileSched"
cap c4_partition "SymSched"
