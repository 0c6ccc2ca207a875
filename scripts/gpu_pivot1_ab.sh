for i in 1 2; do echo "== default"; bash scripts/bench_brief.sh --steps 30 | head -6; echo "== pivot1"; KNN_PIVOT1=1 bash scripts/bench_brief.sh --steps 30 | head -7; done
