#!/bin/bash
# All plans on the headline workload (one bench line each, summarised), then the default
# full bench line (cpu_baseline + e2e) into gpurun_out/bench_full.json.
mkdir -p gpurun_out
make -j8 > /dev/null || exit 1
echo "== default"; bash scripts/bench_brief.sh
echo "== KNN_PIVOT=0"; KNN_PIVOT=0 bash scripts/bench_brief.sh
echo "== KNN_PIVOT=0 KNN_SYM=0"; KNN_PIVOT=0 KNN_SYM=0 bash scripts/bench_brief.sh
echo "== KNN_FUSED=1"; KNN_FUSED=1 bash scripts/bench_brief.sh
timeout -s KILL 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; tail -2 gpurun_out/bench_full.err
python3 -c "
import json; b=json.load(open('gpurun_out/bench_full.json'))
print('full: %.3e pts/s %.3f ms e2e %s cpu %s clocks %s launches %s' % (b['value'], b['ms_per_step'], b['e2e'], b['cpu_baseline'], b['clocks'], b['gpu_launches']))"
