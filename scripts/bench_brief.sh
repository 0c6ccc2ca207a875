#!/bin/bash
# one bench line, summarised (extra args passed to bench.py)
timeout -s KILL 300 python bench.py --no-cpu-baseline --no-e2e "$@" > gpurun_out/bench.json 2>gpurun_out/bench.err || tail -3 gpurun_out/bench.err
python3 -c "
import json; b=json.load(open('gpurun_out/bench.json')); r=b['roofline']
print('%.3e pts/s %.2f ms | %s' % (b['value'], b['ms_per_step'], r['plan']))
for x in [r] + r['others']: print('   %-70s %7.3f ms x%d frac %.3f' % (x['kernel'][:70], x['avg_launch_ms'], x['launches'] // b['steps'], x['frac']))
"
