# Native build: the C-ABI shared library (sm_100a only) and the oracle's C checker.
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3,-pthread --expt-relaxed-constexpr
PKG := paper_1210_7292_b200
SRC := $(wildcard $(PKG)/csrc/*.cu)
OBJ := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(SRC))
HDR := $(wildcard $(PKG)/csrc/*.cuh $(PKG)/csrc/*.hpp) include/chebm2l.h

PYINC := $(shell python3 -c "import sysconfig; print(sysconfig.get_paths()['include'])")

all: $(PKG)/libchebm2l.so $(PKG)/libcfm_batch.so

# reference batch (Python objects) -> CSR, in C (loaded with ctypes.PyDLL)
$(PKG)/libcfm_batch.so: $(PKG)/csrc/batch_csr.cpp include/chebm2l_batch.h
	g++ -O3 -std=c++17 -shared -fPIC -pthread -I$(PYINC) -o $@ $<

# one object per translation unit (make -j builds them in parallel)
build/%.o: $(PKG)/csrc/%.cu $(HDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c -o $@ $<

$(PKG)/libchebm2l.so: $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ) -lcudart

ptxas: $(SRC) $(HDR)
	for f in $(SRC); do $(NVCC) $(NVFLAGS) -Xptxas -v -c -o /tmp/ptxas.o $$f 2>&1 | grep -E "Compiling|registers|spill"; done

sass: $(PKG)/libchebm2l.so
	/usr/local/cuda/bin/cuobjdump -sass $< | grep -oE "DMMA[.0-9x]*|LDGSTS[.A-Z0-9]*" | sort | uniq -c

clean:
	rm -f $(PKG)/libchebm2l.so $(PKG)/libcfm_batch.so build/*.o

.PHONY: all ptxas sass clean
