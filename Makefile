# Builds libvrg.so (sm_100a CUDA kernels + C ABI, in-tree) and the oracle (reference + shim).
NVCC      ?= /usr/local/cuda/bin/nvcc
CUDA_HOME ?= /usr/local/cuda
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall --expt-relaxed-constexpr \
             -Xptxas -warn-spills
PKG       := paper_1604_02153_b200
SRC       := $(PKG)/csrc
BUILD     := $(PKG)/build
CU        := runtime interp spectral transport heun inverse precond batch cabi
OBJS      := $(addprefix $(BUILD)/,$(addsuffix .o,$(CU)))
HDRS      := $(wildcard $(SRC)/*.cuh) include/vrg.h

all: $(PKG)/libvrg.so oracle

$(BUILD):
	mkdir -p $(BUILD)

$(BUILD)/%.o: $(SRC)/%.cu $(HDRS) | $(BUILD)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(PKG)/libvrg.so: $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -L$(CUDA_HOME)/lib64 -lcufft -lcudart

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf $(BUILD) $(PKG)/libvrg.so
	$(MAKE) -C oracle clean

.PHONY: all oracle clean
