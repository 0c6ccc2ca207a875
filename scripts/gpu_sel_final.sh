#!/bin/bash
# two-pass select: parity, timings vs the one-pass kernel, ncu at the headline row length
mkdir -p gpurun_out
make -j16 > /dev/null || exit 1
timeout -s KILL 900 python -m pytest tests/test_gpu_select.py -m gpu -x -q 2>&1 | tail -2
C="16384,65536,32 8192,131072,32 32768,16384,32 65536,8192,32 32768,8192,16 65536,4096,32 65536,4096,1 131072,2048,16 131072,1024,8"
echo "== two-pass"; timeout -s KILL 300 python scripts/select_bench.py $C
echo "== one-pass (KNN_SELECT_ONEPASS=1)"; KNN_SELECT_ONEPASS=1 timeout -s KILL 300 python scripts/select_bench.py $C
for cfg in "n65536 16384,65536,32" "n4096 65536,4096,32"; do set -- $cfg
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k "regex:select" -s 1 -c 1 \
     -o gpurun_out/r02_sel_$1 -f python scripts/select_bench.py $2 > /dev/null 2>&1
done
