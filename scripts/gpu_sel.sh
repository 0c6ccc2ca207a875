#!/bin/bash
# Select parity tests (+ optionally the whole GPU suite) and the C4 (k=1024) bench line.
mkdir -p gpurun_out
make -j8 > /dev/null || exit 1
timeout -s KILL 900 python -m pytest ${TESTS:-tests/test_gpu_select.py} -x -q 2>&1 | tail -5
bash scripts/bench_brief.sh --config C4 --steps 5
