#!/bin/bash
# bench A/B over the builds named as args (ablibs/<name>.so), then quick parity of the last one
for i in 1 2; do for v in "$@"; do echo "== $v"; KNN_LIB_PATH=ablibs/$v.so bash scripts/bench_brief.sh --steps 30 | head -2; done; done
bash scripts/gpu_epi_ab.sh "$@"
