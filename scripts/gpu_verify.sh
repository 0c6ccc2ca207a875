#!/bin/bash
# Full verification pass: GPU parity suite, smoke, full bench line (cpu_baseline + e2e).
mkdir -p gpurun_out
make -j8 > /dev/null || exit 1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -8 | tee gpurun_out/pytest_gpu.txt
timeout -s KILL 300 python __graft_entry__.py smoke 2>&1 | tail -2
timeout -s KILL 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; tail -2 gpurun_out/bench_full.err
cat gpurun_out/bench_full.json
