#!/bin/bash
# A/B of the symmetric schedule order (KNN_SYM_GROUP rows per group; 0 = row-major).
make -j8 > /dev/null || exit 1
for cfg in H C4 C5; do
  for g in 0 8 16; do echo "== $cfg group $g"; KNN_SYM_GROUP=$g bash scripts/bench_brief.sh --config $cfg --steps 5 | head -2; done
done
