#!/bin/bash
# GPU iteration: build, the named test files (default: all GPU tests), then one bench line.
#   TESTS="tests/test_gpu_sharded.py tests/test_gpu_bench.py" bash scripts/gpu_tests.sh
mkdir -p gpurun_out
make -j16 > gpurun_out/make.log 2>&1 || { tail -20 gpurun_out/make.log; exit 1; }
timeout -s KILL ${TEST_TIMEOUT:-1500} python -m pytest ${TESTS:-tests} -m gpu -x -q ${PYTEST_ARGS} 2>&1 | tail -${TAIL:-25}
if [ -z "$NO_BENCH" ]; then
  timeout -s KILL 600 python bench.py ${BENCH_ARGS:---steps 20 --warmup 5 --no-cpu-baseline} > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
  python3 scripts/bench_summary.py gpurun_out/bench.json
fi
