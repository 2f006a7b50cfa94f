# Builds the B200 library (CUDA kernels + C ABI), the C++ drop-in host
# library, the dfakit CLI and the test-only oracle.
#   make            -> paper_2508_20735_b200/lib/libdfakit_b200.so, bin/dfakit, oracle/
NVCC     ?= /usr/local/cuda/bin/nvcc
CXX      ?= g++
ARCH     := -gencode arch=compute_100a,code=sm_100a
NVFLAGS  := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude -Ipaper_2508_20735_b200/csrc \
            --expt-relaxed-constexpr -Xptxas -v
CXXFLAGS := -O2 -fPIC -std=c++20 -Iinclude -Wall -Wextra -Wno-unused-parameter
PKG      := paper_2508_20735_b200
CSRC     := $(PKG)/csrc
BUILD    := build
LIB      := $(PKG)/lib/libdfakit_b200.so
CU_SRCS  := $(wildcard $(CSRC)/*.cu)
CU_OBJS  := $(patsubst $(CSRC)/%.cu,$(BUILD)/%.o,$(CU_SRCS))
HOST_SRCS:= $(wildcard $(CSRC)/host/*.cpp)
HOST_OBJS:= $(patsubst $(CSRC)/host/%.cpp,$(BUILD)/host_%.o,$(HOST_SRCS))

all: $(LIB) bin/dfakit oracle refsuites

$(BUILD)/%.o: $(CSRC)/%.cu $(wildcard $(CSRC)/*.cuh) include/dfakit_b200.h
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(BUILD)/$*.ptxas.log || (cat $(BUILD)/$*.ptxas.log; false)

$(BUILD)/host_%.o: $(CSRC)/host/%.cpp $(wildcard include/dfakit/*.hpp) include/dfakit_b200.h include/dfakit_b200.hpp
	@mkdir -p $(BUILD)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(LIB): $(CU_OBJS) $(HOST_OBJS)
	@mkdir -p $(PKG)/lib
	$(NVCC) $(ARCH) -shared -o $@ $^ -Xcompiler -fPIC -lcudart_static -lpthread -ldl -lrt

bin/dfakit: $(CSRC)/cli/dfakit_cli.cpp $(LIB) include/dfakit_b200.hpp
	@mkdir -p bin
	$(CXX) $(CXXFLAGS) -o $@ $< -L$(PKG)/lib -ldfakit_b200 -Wl,-rpath,'$$ORIGIN/../$(PKG)/lib' -lpthread

oracle:
	$(MAKE) -s -C oracle

# the reference's own unit suites + acceptance harness, compiled unchanged
# against include/ and the library (needs /root/reference; no-op without it)
refsuites: $(LIB) bin/dfakit
	$(MAKE) -s -C tests/refsuites

# tuning experiments: make variant V=name DEFS="-DDFAKIT_X=Y" builds
# $(PKG)/lib/variants/libdfakit_b200_name.so (loaded with DFAKIT_LIB_VARIANT=name)
VOBJS = $(patsubst $(CSRC)/%.cu,$(BUILD)/v_$(V)/%.o,$(CU_SRCS))
$(BUILD)/v_$(V)/%.o: $(CSRC)/%.cu $(wildcard $(CSRC)/*.cuh) include/dfakit_b200.h
	@mkdir -p $(BUILD)/v_$(V)
	$(NVCC) $(NVFLAGS) $(DEFS) -c $< -o $@ 2> $(BUILD)/v_$(V)/$*.ptxas.log || (cat $(BUILD)/v_$(V)/$*.ptxas.log; false)
variant: $(VOBJS) $(HOST_OBJS)
	@mkdir -p $(PKG)/lib/variants
	$(NVCC) $(ARCH) -shared -o $(PKG)/lib/variants/libdfakit_b200_$(V).so $^ -Xcompiler -fPIC -lcudart_static -lpthread -ldl -lrt

clean:
	rm -rf $(BUILD) $(PKG)/lib bin
	$(MAKE) -s -C oracle clean
	$(MAKE) -s -C tests/refsuites clean

.PHONY: all oracle refsuites clean variant
