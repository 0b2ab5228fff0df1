# Builds the in-tree C-ABI library for B200 (sm_100a) and the oracle checker.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall --expt-relaxed-constexpr $(EXTRA)
PKG := paper_2308_02494_b200
SRCS := $(wildcard $(PKG)/csrc/*.cu)
OBJS := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(SRCS))
HDRS := $(wildcard $(PKG)/csrc/*.cuh) include/apmg_cuda.h
LIB := $(PKG)/libapmg_cuda.so

all: $(LIB)

build/%.o: $(PKG)/csrc/%.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -Xptxas -v -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; exit 1)

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcudart

clean:
	rm -rf build $(LIB)

.PHONY: all clean
