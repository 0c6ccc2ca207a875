#!/bin/bash
# Quick GPU iteration: parity tests then the bench line.
mkdir -p gpurun_out
make -j8 > /dev/null || exit 1
timeout -s KILL 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout -s KILL 600 python bench.py ${BENCH_ARGS:---no-cpu-baseline} > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
python3 -c "
import json; b=json.load(open('gpurun_out/bench.json')); r=b['roofline']
print('value %.3e pts/s  ms/step %.2f  e2e %s  plan %s' % (b['value'], b['ms_per_step'], b['e2e'] and '%.3e'%b['e2e']['value'], r['plan']))
print('dominant', r['kernel'], 'avg %.3f ms frac %.3f achieved %.1f %s' % (r['avg_launch_ms'], r['frac'], r['achieved'], r['unit']))
for o in r['others']: print('other', o['kernel'], 'avg %.3f ms frac %.3f achieved %.1f %s' % (o['avg_launch_ms'], o['frac'], o['achieved'], o['unit']))
print('share', r['step_share'], 'clocks', b['clocks'], 'cpu', b['cpu_baseline'] and b['cpu_baseline']['value'])
"
