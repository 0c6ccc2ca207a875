#!/bin/bash
# round-2 batch: tests of the changed paths, bench, sanitizer re-check, select ring variants
make -j16 > /dev/null || exit 1
timeout -s KILL 1500 python -m pytest tests/test_gpu_knn.py tests/test_gpu_select.py tests/test_gpu_sharded.py tests/test_gpu_random.py -m gpu -x -q 2>&1 | tail -6
timeout -s KILL 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err
python3 scripts/bench_summary.py gpurun_out/bench.json
for v in s3w4 s4w4 s6w4 s3w8 s4w2; do echo "== sel $v"; KNN_LIB_PATH=ablibs/sel_$v.so timeout 300 python scripts/select_bench.py 65536,65536,32 16384,65536,1 8192,8192,64 32768,4096,32 65536,8192,16; done
TOOLS="racecheck synccheck" CASES="c1 pivot selects" SAN_TIMEOUT=600 bash scripts/sanitize.sh
