# Build the sm_100a C-ABI library in-tree (travels to the GPU box with gpurun).
NVCC ?= nvcc
PKG := paper_2510_27191_b200
SRC := $(PKG)/csrc/vp_kernels.cu
HDR := $(wildcard $(PKG)/csrc/*.cuh) include/vpb200.h
LIB := $(PKG)/libvpb200.so
# -fmad=false: no FMA contraction, so fp64 arithmetic rounds exactly like the
# numpy reference (parity mode) -- the path is memory bound, FMAs buy nothing.
NVFLAGS := -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
           -fmad=false -Xcompiler -fPIC,-O2 -Xptxas -v --expt-relaxed-constexpr

all: $(LIB)

$(LIB): $(SRC) $(HDR)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRC) 2> build_ptxas.log || (cat build_ptxas.log; exit 1)

clean:
	rm -f $(LIB) build_ptxas.log

.PHONY: all clean
