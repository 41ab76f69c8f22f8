# Builds the sm_100a C-ABI library in-tree (it travels to the GPU box with the
# repo snapshot) and the oracle's C restatement.
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v
PKG := paper_1208_1975_b200
SRCS := $(wildcard $(PKG)/csrc/*.cu)
HDRS := $(wildcard $(PKG)/csrc/*.cuh) include/psmooth.h

all: $(PKG)/libpsmooth.so oracle

$(PKG)/libpsmooth.so: $(SRCS) $(HDRS)
	$(NVCC) $(NVFLAGS) -shared -Xlinker --no-undefined -o $@ $(SRCS) -lcublas -lcudart 2> build_ptxas.log || (cat build_ptxas.log; exit 1)

oracle:
	$(MAKE) -C oracle

clean:
	rm -f $(PKG)/libpsmooth.so build_ptxas.log
	$(MAKE) -C oracle clean

.PHONY: all oracle clean
