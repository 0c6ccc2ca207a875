#!/bin/bash
# A-resident sample pass vs the streamed one (KNN_MINS_RESIDENT=0); then the pivot-plan tests
make -j16 > /dev/null || exit 1
for i in 1 2; do for r in 0 1; do echo "== mins resident $r"; KNN_MINS_RESIDENT=$r bash scripts/bench_brief.sh --steps 30 | head -6; done; done
for d in 12 16; do echo "== pivot_div $d"; KNN_PIVOT_DIV=$d bash scripts/bench_brief.sh --steps 30 | head -6; done
timeout -s KILL 1800 python -m pytest tests/test_gpu_knn.py tests/test_gpu_random.py tests/test_gpu_sharded.py tests/test_gpu_cosine.py -m gpu -x -q 2>&1 | tail -3
