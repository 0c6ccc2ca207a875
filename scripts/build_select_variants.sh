#!/bin/bash
# A/B builds of the warp-per-row select's ring (stages / warps per CTA): ablibs/sel_<tag>.so
set -e
make -j16 > /dev/null
NCCL_DIR=$(python3 -c "import nvidia.nccl as m; print(list(m.__path__)[0])")
FL="-std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC --expt-relaxed-constexpr -I$NCCL_DIR/include"
OBJS=$(ls build/*.o | grep -v select.o)
mkdir -p ablibs
for v in "s3w4:-DKNN_WSEL_S=3 -DKNN_WSEL_WARPS=4" "s4w4:-DKNN_WSEL_S=4 -DKNN_WSEL_WARPS=4" "s6w4:-DKNN_WSEL_S=6 -DKNN_WSEL_WARPS=4" "s3w8:-DKNN_WSEL_S=3 -DKNN_WSEL_WARPS=8" "s4w2:-DKNN_WSEL_S=4 -DKNN_WSEL_WARPS=2"; do
  tag=${v%%:*}; defs=${v#*:}
  nvcc $FL $defs -c paper_1309_5478_b200/csrc/select.cu -o /tmp/sel_$tag.o
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ablibs/sel_$tag.so $OBJS /tmp/sel_$tag.o -lcudart -ldl
  echo built $tag
done
