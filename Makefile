# Native build: the C-ABI shared library (sm_100a only) and the oracle's C checker.
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3,-pthread --expt-relaxed-constexpr
PKG := paper_1210_7292_b200
SRC := $(PKG)/csrc/capi.cu
HDR := $(wildcard $(PKG)/csrc/*.cuh $(PKG)/csrc/*.hpp) include/chebm2l.h

all: $(PKG)/libchebm2l.so

$(PKG)/libchebm2l.so: $(SRC) $(HDR)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRC) -lcudart

ptxas: $(SRC) $(HDR)
	$(NVCC) $(NVFLAGS) -Xptxas -v -c -o /tmp/capi.o $(SRC) 2>&1 | grep -E "tile_gemm|registers|spill" | head -40

sass: $(PKG)/libchebm2l.so
	/usr/local/cuda/bin/cuobjdump -sass $< | grep -oE "DMMA[.0-9x]*|LDGSTS[.A-Z0-9]*" | sort | uniq -c

clean:
	rm -f $(PKG)/libchebm2l.so

.PHONY: all ptxas sass clean
