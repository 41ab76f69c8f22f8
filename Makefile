# Builds the sm_100a C-ABI library in-tree (it travels to the GPU box with the
# repo snapshot) and the oracle's C restatement. One object per .cu so that
# `make -j` compiles the translation units in parallel.
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v
PKG := paper_1208_1975_b200
SRCS := $(wildcard $(PKG)/csrc/*.cu)
OBJS := $(patsubst $(PKG)/csrc/%.cu,build/obj/%.o,$(SRCS))
HDRS := $(wildcard $(PKG)/csrc/*.cuh) include/psmooth.h

all: $(PKG)/libpsmooth.so oracle

build/obj/%.o: $(PKG)/csrc/%.cu $(HDRS)
	@mkdir -p build/obj
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> build/obj/$*.ptxas.log || (cat build/obj/$*.ptxas.log; exit 1)

$(PKG)/libpsmooth.so: $(OBJS)
	$(NVCC) $(ARCH) -shared -Xlinker --no-undefined -o $@ $(OBJS) -lcudart
	@cat build/obj/*.ptxas.log > build_ptxas.log

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf $(PKG)/libpsmooth.so build_ptxas.log build/obj
	$(MAKE) -C oracle clean

.PHONY: all oracle clean
