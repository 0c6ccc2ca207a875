mkdir -p gpurun_out
for cfg in "n1024 131072,1024,8" "n4096 65536,4096,32"; do set -- $cfg
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k "regex:select" -s 1 -c 1 \
     -o gpurun_out/sel_${TAG:-v3}_$1 -f python scripts/select_bench.py $2 > /dev/null 2>&1
done
ls gpurun_out
