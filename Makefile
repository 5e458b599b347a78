# B200 build: hand-written sm_100a kernels + host C++ -> in-tree shared library
# paper_2404_16370_b200/lib/libsmcl_gpu.so (C ABI: include/smcl_gpu.h), and the
# CPU oracle (test infrastructure) -> oracle/build/libsmcl_oracle.so.
NVCC ?= /usr/local/cuda/bin/nvcc
HOSTCXX := $(shell test -x /usr/bin/g++ && echo /usr/bin/g++ || echo g++)
ARCH := -gencode arch=compute_100a,code=sm_100a
PKG := paper_2404_16370_b200
CSRC := $(PKG)/csrc
BUILD := build/obj
LIB := $(PKG)/lib/libsmcl_gpu.so

# -ffp-contract=off on the host side; device exact paths use __dmul_rn/__dadd_rn.
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++20 -ccbin $(HOSTCXX) --expt-relaxed-constexpr \
           -Xcompiler -fPIC,-ffp-contract=off,-fopenmp -Xptxas -v $(EXTRA_NVFLAGS)
CXXFLAGS := -std=c++20 -O3 -fPIC -fopenmp -ffp-contract=off -Wall -Wextra -Wno-unknown-pragmas

CU_SRC := $(wildcard $(CSRC)/*.cu) $(wildcard $(CSRC)/kernels/*.cu)
CPP_SRC := $(wildcard $(CSRC)/host/*.cpp)
HDRS := $(wildcard $(CSRC)/*.cuh) $(wildcard $(CSRC)/host/*.hpp) include/smcl_gpu.h
CU_OBJ := $(patsubst $(CSRC)/%.cu,$(BUILD)/%.o,$(CU_SRC))
CPP_OBJ := $(patsubst $(CSRC)/%.cpp,$(BUILD)/%.o,$(CPP_SRC))

all: $(LIB) oracle examples/scenario_callsite build/tools/micro_peaks

$(BUILD)/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $@.ptxas.log || (cat $@.ptxas.log; false)

$(BUILD)/%.o: $(CSRC)/%.cpp $(HDRS)
	@mkdir -p $(dir $@)
	$(HOSTCXX) $(CXXFLAGS) -c $< -o $@

# Device scan preparation must round like the -ffp-contract=off host build.
$(BUILD)/kernels/scan_prep.o: NVFLAGS += -fmad=false

$(LIB): $(CU_OBJ) $(CPP_OBJ)
	@mkdir -p $(dir $@)
	$(NVCC) $(ARCH) -shared -ccbin $(HOSTCXX) -o $@ $^ -Xcompiler -fopenmp -lgomp

oracle:
	$(MAKE) -s -C oracle

clean:
	rm -rf build $(PKG)/lib oracle/build

.PHONY: all oracle clean

# Reference-shaped call site compiled against the source-compatible steinmcl:: facade.
examples/scenario_callsite: examples/scenario_callsite.cpp $(wildcard include/steinmcl/*.hpp) include/smcl_gpu.h $(LIB)
	$(HOSTCXX) -std=c++20 -O2 -Wall -Wextra -Iinclude -o $@ examples/scenario_callsite.cpp -L$(PKG)/lib -lsmcl_gpu -Wl,-rpath,'$$ORIGIN/../$(PKG)/lib'

# Roofline microbenchmarks (FP32/FP64 FMA, random record gathers from L2 / HBM).
build/tools/micro_peaks: $(CSRC)/tools/micro_peaks.cu
	@mkdir -p $(dir $@)
	$(NVCC) $(ARCH) -O3 -ccbin $(HOSTCXX) -o $@ $<
