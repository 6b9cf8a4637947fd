# Build libhx.so (sm_100a) in-tree.  `make -j` ; the .so travels to the GPU box with gpurun.
NVCC ?= /usr/local/cuda/bin/nvcc
PKG := paper_1611_09784_b200
SRC := $(wildcard $(PKG)/csrc/*.cu)
HDR := $(wildcard $(PKG)/csrc/*.cuh) include/hx.h
OBJ := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(SRC))
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 --expt-relaxed-constexpr -Xptxas -v -Iinclude

all: $(PKG)/libhx.so

build/%.o: $(PKG)/csrc/%.cu $(HDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(PKG)/libhx.so: $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ) -lpthread

clean:
	rm -rf build $(PKG)/libhx.so

.PHONY: all clean
