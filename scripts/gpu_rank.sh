#!/bin/bash
# adaptive pivot rank vs the certified rank (KNN_PIVOT_RANK=0): bench lines, then GPU tests
make -j16 > /dev/null || exit 1
for i in 1 2; do for r in 0 auto; do echo "== rank $r"; if [ $r = auto ]; then bash scripts/bench_brief.sh --steps 30 | head -6; else KNN_PIVOT_RANK=$r bash scripts/bench_brief.sh --steps 30 | head -6; fi; done; done
for c in C2 C5; do echo "== $c"; bash scripts/bench_brief.sh --config $c --steps 10 | head -3; KNN_PIVOT_RANK=0 bash scripts/bench_brief.sh --config $c --steps 10 | head -1; done
timeout -s KILL 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
