#!/bin/bash
# A/B of select builds in ablibs/ (names as args)
C="16384,65536,32 65536,8192,32 65536,4096,32 131072,2048,16 65536,4096,1 32768,16384,32 8192,131072,32 32768,8192,16 131072,1024,8"
for v in "$@"; do echo "== $v"; KNN_LIB_PATH=ablibs/$v.so timeout -s KILL 300 python scripts/select_bench.py $C; done
