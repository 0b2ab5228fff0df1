# Builds the in-tree C-ABI library for B200 (sm_100a) and, separately, the profiling /
# self-test kernels (tools/csrc -> tools/libapmg_debug.so; never loaded by the package).
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall --expt-relaxed-constexpr $(EXTRA)
PKG := paper_2308_02494_b200
SRCS := $(wildcard $(PKG)/csrc/*.cu)
BUILD ?= build
OBJS := $(patsubst $(PKG)/csrc/%.cu,$(BUILD)/%.o,$(SRCS))
HDRS := $(wildcard $(PKG)/csrc/*.cuh) include/apmg_cuda.h
LIB ?= $(PKG)/libapmg_cuda.so
DBG_SRCS := $(wildcard tools/csrc/*.cu)
DBG_OBJS := $(patsubst tools/csrc/%.cu,build/dbg_%.o,$(DBG_SRCS))
DBG_LIB := tools/libapmg_debug.so

all: $(LIB) $(DBG_LIB)

$(BUILD)/%.o: $(PKG)/csrc/%.cu $(HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -Xptxas -v -c $< -o $@ 2> $(BUILD)/$*.ptxas.log || (cat $(BUILD)/$*.ptxas.log; exit 1)

$(LIB): $(OBJS)
	@mkdir -p $(dir $@)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcudart

build/dbg_%.o: tools/csrc/%.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -I$(PKG)/csrc -c $< -o $@

# the debug kernels use the package's error/launch helpers (runtime.o) statically
$(DBG_LIB): $(DBG_OBJS) build/runtime.o
	$(NVCC) $(ARCH) -shared -o $@ $(DBG_OBJS) build/runtime.o -lcudart

clean:
	rm -rf build $(LIB) $(DBG_LIB)

.PHONY: all clean
