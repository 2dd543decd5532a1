# Build recipe for the B200 product library, the generators and the oracles.
#   make            -> product + generators + C restatement oracle (+ oracle/_ref when /root/reference exists)
#   make product    -> paper_1604_06043_b200/libmstab_b200.so (sm_100a)
#   make ref        -> oracle/_ref/libmstab_ref.so (the unmodified reference, see oracle/Makefile) and the
#                      reference's own GTest suites built against it and against the B200 shim
NVCC ?= /usr/local/cuda/bin/nvcc
CXX ?= g++
CUDA_HOME ?= /usr/local/cuda
PKG := paper_1604_06043_b200
CSRC := $(PKG)/csrc
BUILD := build

ARCH := -gencode arch=compute_100a,code=sm_100a
NVCCFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 --fmad=false -Xcompiler -fPIC -Xptxas -O3
CXXFLAGS := -O3 -std=c++20 -fPIC -ffp-contract=off -Wall -Wextra -I$(CUDA_HOME)/include

HOST_SRCS := $(CSRC)/solver.cpp $(CSRC)/capi.cpp $(CSRC)/host_util.cpp $(CSRC)/comm.cpp
HOST_OBJS := $(patsubst $(CSRC)/%.cpp,$(BUILD)/%.o,$(HOST_SRCS))
CU_SRCS := $(CSRC)/kspmv.cu $(CSRC)/kcdia.cu $(CSRC)/klevel.cu $(CSRC)/kls.cu $(CSRC)/kpoly.cu $(CSRC)/kmisc.cu $(CSRC)/ktri.cu $(CSRC)/ksridr.cu $(CSRC)/kbase.cu
CU_OBJS := $(patsubst $(CSRC)/%.cu,$(BUILD)/%.o,$(CU_SRCS))
HEADERS := $(wildcard $(CSRC)/*.h) $(CSRC)/kcommon.cuh include/mstab_b200.h

all: product gen oracle ref

product: $(PKG)/libmstab_b200.so
gen: $(PKG)/libmstab_gen.so

$(BUILD):
	mkdir -p $(BUILD)

$(BUILD)/%.o: $(CSRC)/%.cu $(HEADERS) | $(BUILD)
	$(NVCC) $(NVCCFLAGS) -c $< -o $@

$(BUILD)/%.o: $(CSRC)/%.cpp $(HEADERS) | $(BUILD)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(PKG)/libmstab_b200.so: $(CU_OBJS) $(HOST_OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $^ -Xlinker -Bsymbolic -lcudart_static -ldl -lrt -lpthread

$(PKG)/libmstab_gen.so: $(CSRC)/generators.cpp include/mstab_gen.h
	$(CXX) $(CXXFLAGS) -shared -o $@ $<

oracle:
	$(MAKE) -C oracle restatement

ref: product
	@if [ -d /root/reference/proj/core/src ]; then $(MAKE) -C oracle ref refsuite shimtests; else echo "reference absent: using prebuilt oracle/_ref"; fi

sass: $(CU_OBJS)
	for o in $(CU_OBJS); do $(CUDA_HOME)/bin/cuobjdump -sass $$o; done > $(BUILD)/kernels.sass

clean:
	rm -rf $(BUILD) $(PKG)/*.so

.PHONY: all product gen oracle ref clean sass
