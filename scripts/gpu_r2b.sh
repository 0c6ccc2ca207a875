#!/bin/bash
# Round-2 re-entry pass: full GPU suite, bench, launch list, select microbench at the
# headline row length and short rows.
mkdir -p gpurun_out
make -j16 > /dev/null || exit 1
timeout -s KILL 1800 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.txt 2>&1; tail -4 gpurun_out/gputests.txt
timeout -s KILL 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err
python3 scripts/bench_summary.py gpurun_out/bench.json
timeout -s KILL 300 python scripts/select_bench.py 16384,65536,32 65536,8192,32 65536,4096,32 131072,2048,16 32768,8192,64 > gpurun_out/selbench.txt 2>&1; cat gpurun_out/selbench.txt
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
grep -v "^==" gpurun_out/r02_launches.csv | python3 -c "import csv,sys,collections; r=list(csv.reader(sys.stdin)); h=r[0]; ki=h.index(\"Kernel Name\"); vi=h.index(\"Metric Value\"); d=collections.defaultdict(list)
for x in r[1:]:
  d[x[ki][:60]].append(float(x[vi].replace(\",\",\"\")))
for k,v in d.items(): print(len(v), round(sum(v)/len(v)/1e3,3),\"us\", k)" 
