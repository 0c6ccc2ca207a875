# sample-size sweep: KNN_PIVOT_DIV (sample = N / div columns) on the headline and C2, C3, C5
make -j16 > /dev/null 2>&1 || exit 1
for dv in ${DIVS:-12 16 24 32}; do echo "== DIV $dv"; KNN_PIVOT_DIV=$dv bash scripts/bench_brief.sh --steps 30 | head -1
  for c in C2 C3 C5; do KNN_PIVOT_DIV=$dv bash scripts/bench_brief.sh --steps 10 --config $c | head -1; done; done
