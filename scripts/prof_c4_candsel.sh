mkdir -p gpurun_out
KNN_CANDSEL_STATS=1 timeout -s KILL 300 python bench.py --config C4 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e 2>&1 | grep candidate_select_warp | head -2
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:candidate_select -s 2 -c 2 \
  -o gpurun_out/c4_candsel -f python bench.py --config C4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/c4_candsel.log 2>&1
tail -3 gpurun_out/c4_candsel.log
