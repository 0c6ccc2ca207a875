#!/bin/bash
# device-chosen single-product partition: GPU tests, bench lines, calibration on C2/C5
make -j16 > /dev/null || exit 1
for c in H C2 C5 C3; do for p in "" 0 1; do echo "== $c KNN_PIVOT1=$p"; if [ -z "$p" ]; then unset KNN_PIVOT1; else export KNN_PIVOT1=$p; fi; A=""; [ $c != H ] && A="--config $c"; bash scripts/bench_brief.sh --steps 20 $A | head -3; done; unset KNN_PIVOT1; done
timeout -s KILL 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
