#!/bin/bash
# compute-sanitizer over the small cases of scripts/sanitize_cases.py; logs -> gpurun_out/san_*.txt
mkdir -p gpurun_out
make -j16 > /dev/null || exit 1
for tool in ${TOOLS:-memcheck racecheck synccheck initcheck}; do
  for c in ${CASES:-c1 pivot pivotq selects par3}; do
    timeout -s KILL ${SAN_TIMEOUT:-900} compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 \
      python scripts/sanitize_cases.py $c > gpurun_out/san_${tool}_${c}.txt 2>&1
    echo "$tool $c rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san_${tool}_${c}.txt | tail -1)"
  done
done
