# Build libknn.so (sm_100a) and the CPU oracle.  `make` or __graft_entry__.build().
NVCC      ?= nvcc
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := -std=c++17 -O3 -lineinfo $(ARCH) -Xcompiler -fPIC -Xcompiler -Wall $(NVFLAGS_EXTRA) \
             -Xptxas -v --expt-relaxed-constexpr
# NCCL: header from the torch-bundled wheel (types only); the library is dlopen'ed at run
# time (libnccl.so.2, falling back to this wheel's copy)
NCCL_DIR  ?= $(shell python3 -c "import nvidia.nccl as m; print(list(m.__path__)[0])" 2>/dev/null)
NVFLAGS   += -I$(NCCL_DIR)/include -DKNN_NCCL_LIB='"$(NCCL_DIR)/lib/libnccl.so.2"'
SRC_DIR   := paper_1309_5478_b200/csrc
BUILD     := build
SRCS      := $(wildcard $(SRC_DIR)/*.cu)
OBJS      := $(patsubst $(SRC_DIR)/%.cu,$(BUILD)/%.o,$(SRCS))
LIB       := paper_1309_5478_b200/libknn.so
ORACLE    := oracle/liboracle.so

all: $(LIB) $(ORACLE)

$(BUILD)/%.o: $(SRC_DIR)/%.cu $(SRC_DIR)/internal.cuh $(SRC_DIR)/ptx.cuh $(SRC_DIR)/tc_common.cuh $(SRC_DIR)/warpsel.cuh $(SRC_DIR)/runtime.h include/knn.h
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(BUILD)/$*.ptxas.log || (cat $(BUILD)/$*.ptxas.log; exit 1)

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcudart -ldl

$(ORACLE): oracle/knn_oracle.cpp
	g++ -O2 -ffp-contract=off -std=c++17 -shared -fPIC -pthread -o $@ $<

clean:
	rm -rf $(BUILD) $(LIB) $(ORACLE)

.PHONY: all clean
