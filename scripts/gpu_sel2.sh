#!/bin/bash
# two-pass warp select: parity (select tests) and timing against the one-pass warp select
mkdir -p gpurun_out
make -j16 > /dev/null || exit 1
python scripts/dbg_sel2.py
timeout -s KILL 900 python -m pytest tests/test_gpu_select.py -m gpu -x -q 2>&1 | tail -4
C="16384,65536,32 65536,8192,32 65536,4096,32 131072,2048,16 65536,4096,1 32768,16384,32 8192,131072,32 32768,8192,16 131072,1024,8"
echo "== two-pass"; timeout -s KILL 300 python scripts/select_bench.py $C
for st in 2 4 6; do echo "== two-pass stages $st"; KNN_WS2_STAGES=$st timeout -s KILL 300 python scripts/select_bench.py 16384,65536,32 65536,4096,32 131072,2048,16; done
echo "== one-pass"; KNN_SELECT_ONEPASS=1 timeout -s KILL 300 python scripts/select_bench.py $C
