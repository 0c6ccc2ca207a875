timeout -s KILL 900 python -m pytest tests/test_gpu_select.py -m gpu -x -q -k "two_pass or warp" 2>&1 | tail -2
bash scripts/gpu_selab.sh contig pre1
for cfg in "n65536 16384,65536,32" "n4096 65536,4096,32"; do set -- $cfg
timeout -s KILL 600 ncu --metrics dram__bytes_read.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum -k "regex:select" -s 1 -c 1 python scripts/select_bench.py $2 2>&1 | grep -E "dram__|lts__|gpu__time"
done
