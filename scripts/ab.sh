#!/bin/bash
# A/B of two library builds on the same box: ablibs/old.so vs build/ab/new.so, alternating.
for i in 1 2 3; do
  for v in old new; do echo "== $v"; KNN_LIB_PATH=ablibs/$v.so bash scripts/bench_brief.sh --steps 30 ${BENCH_ARGS} | head -2; done
done
