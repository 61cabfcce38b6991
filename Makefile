# Builds the CUDA product library (sm_100a) and the CPU oracle.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 -Xptxas -v
PKG := paper_1703_00640_b200
SRC := $(wildcard $(PKG)/csrc/*.cu) $(PKG)/csrc/params.cpp
HDR := $(wildcard $(PKG)/csrc/*.cuh) $(wildcard $(PKG)/csrc/*.hpp) include/truncmul_b200.h
LIB := $(PKG)/libtruncmul_b200.so

all: $(LIB) oracle

$(LIB): $(SRC) $(HDR)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRC) 2> build_ptxas.log || (cat build_ptxas.log; exit 1)

oracle:
	$(MAKE) -C oracle

clean:
	rm -f $(LIB) build_ptxas.log
	$(MAKE) -C oracle clean

.PHONY: all oracle clean
