#!/bin/bash
# e2e A/B: pipelined k-NNG chunk divisor (KNN_PIPE_DIV), probe timings
mkdir -p gpurun_out
make -j16 > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_knn.py -m gpu -x -q -k "host" 2>&1 | tail -2
for dv in 8 16 32; do echo "== KNN_PIPE_DIV=$dv"; KNN_PIPE_DIV=$dv timeout 300 python scripts/e2e_probe.py 2>&1 | tail -2; done
for dv in 8 16; do
  KNN_PIPE_DIV=$dv timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline > gpurun_out/b_e2e.json 2>/dev/null
  python3 -c "import json; b=json.load(open('gpurun_out/b_e2e.json')); print('DIV $dv value %.3e e2e %.3e' % (b['value'], b['e2e']['value']))"
done
