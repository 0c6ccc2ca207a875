#!/bin/bash
# GPU iteration: build, selected tests (TESTS, KEXPR), the headline brief bench (with the
# re-evaluation set size), then the configs C2..C5 (CONFIGS=0 skips them).
mkdir -p gpurun_out
make -j16 > gpurun_out/make.log 2>&1 || { tail -20 gpurun_out/make.log; exit 1; }
if [ -n "$TESTS" ]; then
  timeout -s KILL ${TEST_TIMEOUT:-1200} python -m pytest $TESTS -m gpu -x -q ${KEXPR:+-k "$KEXPR"} 2>&1 | tail -${TAIL:-15}
fi
echo "== H default"; bash scripts/bench_brief.sh --steps 30
echo "== H KNN_PIVOT1=0"; KNN_PIVOT1=0 bash scripts/bench_brief.sh --steps 30
KNN_RECOMP_STATS=1 timeout 120 python -c "
import torch
from paper_1309_5478_b200 import knn, datagen
X = torch.from_numpy(datagen.points(65536, 256, 'uniform', seed=1)).cuda()
knn.graph(X, 32); print('|R| per row (re-evaluated):', knn.last_candidates() / 65536, 'plan', knn.last_plan())
"
timeout 120 python -c "
import torch
from paper_1309_5478_b200 import knn, datagen
X = torch.from_numpy(datagen.points(65536, 256, 'uniform', seed=1)).cuda()
knn.graph(X, 32); print('candidates per row:', knn.last_candidates() / 65536, 'plan', knn.last_plan())
"
if [ "${CONFIGS:-1}" = "1" ]; then
  for c in C2 C3 C4 C5; do echo "== config $c"; bash scripts/bench_brief.sh --config $c --steps 10; done
fi
