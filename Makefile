# Builds the C-ABI library for B200 (sm_100a).  `python -c "import __graft_entry__ as g; g.build()"` does the same.
NVCC ?= /usr/local/cuda/bin/nvcc
PKG := paper_2003_07065_b200
SRC := $(PKG)/csrc/sst_api.cu $(PKG)/csrc/sst_kernels.cu $(PKG)/csrc/ridge.cu $(PKG)/csrc/multipass.cu
HDR := include/sst.h $(PKG)/csrc/sst_internal.h $(PKG)/csrc/fft.cuh $(PKG)/csrc/decide.cuh
FLAGS := -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 -shared \
         -Xptxas -v -cudart static

$(PKG)/libsst.so: $(SRC) $(HDR)
	$(NVCC) $(FLAGS) -o $@ $(SRC) 2> build_ptxas.log || (cat build_ptxas.log; exit 1)

clean:
	rm -f $(PKG)/libsst.so build_ptxas.log
.PHONY: clean
