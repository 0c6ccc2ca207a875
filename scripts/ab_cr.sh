#!/bin/bash
# A/B of the re-evaluation kernel's CTAs per SM (KNN_CR_MINB) and T subset (KNN_CR_T)
mkdir -p gpurun_out
for v in ${VARIANTS:-"-DKNN_CR_MINB=4" "-DKNN_CR_MINB=5" "-DKNN_CR_MINB=6"}; do
  touch paper_1309_5478_b200/csrc/select.cu
  make -j16 NVFLAGS_EXTRA="$v" > gpurun_out/make_ab.log 2>&1 || { echo build failed; tail gpurun_out/make_ab.log; exit 1; }
  grep -A2 "candidate_recompute" build/select.ptxas.log | grep -E "spill|Used" | tr '\n' ' '; echo
  echo "== $v"; bash scripts/bench_brief.sh --steps 40 | grep -E "pts/s|recompute"
done
touch paper_1309_5478_b200/csrc/select.cu; make -j16 > /dev/null 2>&1
