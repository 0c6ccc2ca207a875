# single-product partition (KNN_PIVOT1=1) vs the default 3-product partition, vs the oracle
for cfg in "65536 256 32 0" "65536 256 32 1" "20000 48 10 0 gauss" "32768 64 16 1 clusters"; do
  KNN_PIVOT1=1 timeout 300 python scripts/pivot1_check.py $cfg 2>&1 | tail -1
  timeout 300 python scripts/pivot1_check.py $cfg 2>&1 | tail -1
done
