#!/bin/bash
# pivot sample size sweep (KNN_PIVOT_DIV): step and per-kernel times
make -j16 > /dev/null || exit 1
for i in 1 2; do for d in 8 4 16 6; do echo "== pivot_div $d"; KNN_PIVOT_DIV=$d bash scripts/bench_brief.sh --steps 30 | head -6; done; done
