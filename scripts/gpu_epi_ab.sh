#!/bin/bash
# partition time with parts of the epilogue disabled (KNN_DBG_EPI), for the builds named as args
for v in "$@"; do for d in 0 4 2 16 8; do echo -n "$v "; KNN_LIB_PATH=ablibs/$v.so KNN_DBG_EPI=$d timeout 120 python scripts/epi_cost.py 2>&1 | tail -1; done; done
