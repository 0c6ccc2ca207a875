#!/bin/bash
# One bench line per config (C1..C5 on one GPU) and per plan on the headline.
mkdir -p gpurun_out
make -j8 > /dev/null || exit 1
for c in C1 C2 C3 C4 C5; do echo "== config $c"; bash scripts/bench_brief.sh --config $c --steps 10; cp gpurun_out/bench.json gpurun_out/bench_$c.json; done
echo "== H default"; bash scripts/bench_brief.sh
echo "== H KNN_PIVOT1=0 (3-product partition)"; KNN_PIVOT1=0 bash scripts/bench_brief.sh
echo "== H KNN_PIVOT=0"; KNN_PIVOT=0 bash scripts/bench_brief.sh
echo "== H KNN_PIVOT=0 KNN_SYM=0"; KNN_PIVOT=0 KNN_SYM=0 bash scripts/bench_brief.sh
