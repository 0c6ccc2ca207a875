mkdir -p gpurun_out
make -j8 > /dev/null || exit 1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:select_ring -s 2 -c 1 \
  -o gpurun_out/c4_select -f python bench.py --config C4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/c4_select.log 2>&1
tail -3 gpurun_out/c4_select.log
