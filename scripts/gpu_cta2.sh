#!/bin/bash
# cta_group::2 mainloop: quick correctness, then bench lines vs the 1-CTA build (ablibs/cta1.so)
make -j16 > /dev/null || exit 1
timeout -s KILL 300 python -m pytest tests/test_gpu_knn.py -m gpu -x -q -k "distances or c1_graph or symmetric or headline or pivot_graph_equals" 2>&1 | tail -3
for i in 1 2; do for v in cta1 cta2; do echo "== $v"; KNN_LIB_PATH=ablibs/$v.so bash scripts/bench_brief.sh --steps 30 | head -6; done; done
