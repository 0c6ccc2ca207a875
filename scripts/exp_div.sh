# sample-size sweep: KNN_PIVOT_DIV (sample = N / div columns), interleaved repetitions
make -j16 > /dev/null 2>&1 || exit 1
for rep in 1 2 3; do for dv in ${DIVS:-8 12 16}; do
  echo "== DIV $dv rep $rep $(KNN_PIVOT_DIV=$dv bash scripts/bench_brief.sh --steps 60 | head -1 | cut -c1-30) C5 $(KNN_PIVOT_DIV=$dv bash scripts/bench_brief.sh --steps 10 --config C5 | head -1 | cut -c1-30) C3 $(KNN_PIVOT_DIV=$dv bash scripts/bench_brief.sh --steps 10 --config C3 | head -1 | cut -c1-30)"
done; done
