#!/bin/bash
# A/B of the single-product partition's epilogue warps (KNN_PV1_WARPS 16 / 20)
mkdir -p gpurun_out
for w in ${WARPSETS:-20 16 20 16}; do
  touch paper_1309_5478_b200/csrc/gemm_tc.cu
  make -j16 NVFLAGS_EXTRA="-DKNN_PV1_WARPS=$w" > gpurun_out/make_ab.log 2>&1 || { echo build failed; tail gpurun_out/make_ab.log; exit 1; }
  echo "== KNN_PV1_WARPS=$w $(bash scripts/bench_brief.sh --steps 40 | grep -E 'pts/s|PIVOT1' | tr -s ' ' | cut -c1-120 | tr '\n' ' ')"
  echo "   C5 $(bash scripts/bench_brief.sh --steps 10 --config C5 | head -1 | cut -c1-30)  C3 $(bash scripts/bench_brief.sh --steps 10 --config C3 | head -1 | cut -c1-30)"
done
if [ -n "$TEST20" ]; then
  touch paper_1309_5478_b200/csrc/gemm_tc.cu; make -j16 NVFLAGS_EXTRA="-DKNN_PV1_WARPS=20" > /dev/null 2>&1
  timeout 900 python -m pytest tests/test_gpu_knn.py tests/test_gpu_random.py tests/test_gpu_sharded.py -m gpu -x -q -k "pivot or host or per_point or full_size or random or sym or auto" 2>&1 | tail -2
fi
touch paper_1309_5478_b200/csrc/gemm_tc.cu; make -j16 > /dev/null 2>&1
