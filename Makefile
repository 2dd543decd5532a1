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

HOST_SRCS := $(CSRC)/solver.cpp $(CSRC)/capi.cpp $(CSRC)/host_util.cpp $(CSRC)/comm.cpp $(CSRC)/zsolver.cpp
HOST_OBJS := $(patsubst $(CSRC)/%.cpp,$(BUILD)/%.o,$(HOST_SRCS))
CU_SRCS := $(CSRC)/kspmv.cu $(CSRC)/kcdia.cu $(CSRC)/klevel.cu $(CSRC)/kls.cu $(CSRC)/kpoly.cu $(CSRC)/kmisc.cu $(CSRC)/ktri.cu $(CSRC)/ksridr.cu $(CSRC)/kbase.cu $(CSRC)/kpersist.cu $(CSRC)/kcomplex.cu
CU_OBJS := $(patsubst $(CSRC)/%.cu,$(BUILD)/%.o,$(CU_SRCS))
HEADERS := $(wildcard $(CSRC)/*.h) $(CSRC)/kcommon.cuh $(CSRC)/kdense.cuh $(CSRC)/ktimeline.cuh include/mstab_b200.h include/mstab_b200_kernels.h

all: product gen oracle ref

product: $(PKG)/libmstab_b200.so
gen: $(PKG)/libmstab_gen.so

$(BUILD):
	mkdir -p $(BUILD)

$(BUILD)/%.o: $(CSRC)/%.cu $(HEADERS) | $(BUILD)
	$(NVCC) $(NVCCFLAGS) -c $< -o $@

$(BUILD)/%.o: $(CSRC)/%.cpp $(HEADERS) | $(BUILD)
	$(CXX) $(CXXFLAGS) -c $< -o $@

# build provenance (mstab_build_id): git HEAD, a content hash of every product source and the
# nvcc flags; rewritten only when it changes, so capi.o rebuilds exactly when the id does
$(BUILD)/build_id.h: FORCE | $(BUILD)
	@printf '#define MSTAB_GIT_SHA "%s src:%s"\n#define MSTAB_BUILD_FLAGS "nvcc %s"\n' \
	  "$$(git rev-parse --short=12 HEAD 2>/dev/null || echo nogit)$$(git diff --quiet HEAD -- $(CSRC) include Makefile 2>/dev/null || echo -dirty)" \
	  "$$(cat $(HOST_SRCS) $(CU_SRCS) $(HEADERS) | sha256sum | cut -c1-12)" "$(NVCCFLAGS)" > $@.tmp
	@cmp -s $@.tmp $@ || mv $@.tmp $@; rm -f $@.tmp

$(BUILD)/capi.o: $(CSRC)/capi.cpp $(HEADERS) $(BUILD)/build_id.h | $(BUILD)
	$(CXX) $(CXXFLAGS) -include $(BUILD)/build_id.h -c $< -o $@

$(PKG)/libmstab_b200.so: $(CU_OBJS) $(HOST_OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $^ -Xlinker -Bsymbolic -lcudart_static -ldl -lrt -lpthread

$(PKG)/libmstab_gen.so: $(CSRC)/generators.cpp include/mstab_gen.h
	$(CXX) $(CXXFLAGS) -shared -o $@ $<

oracle:
	$(MAKE) -C oracle restatement

ref: product
	@if [ -d /root/reference/proj/core/src ]; then $(MAKE) -C oracle ref refsuite shimtests; else echo "reference absent: using prebuilt oracle/_ref"; fi

# developer build with the ktimeline.cuh probes compiled in (tools/timeline.py loads it)
TL_BUILD := build/tl
TL_OBJS := $(patsubst $(CSRC)/%.cu,$(TL_BUILD)/%.o,$(CU_SRCS)) $(patsubst $(CSRC)/%.cpp,$(TL_BUILD)/%.o,$(HOST_SRCS))
timeline: $(PKG)/libmstab_b200_tl.so
$(TL_BUILD)/%.o: $(CSRC)/%.cu $(HEADERS) $(CSRC)/ktimeline.cuh
	@mkdir -p $(TL_BUILD)
	$(NVCC) $(NVCCFLAGS) -DMSTAB_TIMELINE -c $< -o $@
$(TL_BUILD)/%.o: $(CSRC)/%.cpp $(HEADERS) $(BUILD)/build_id.h
	@mkdir -p $(TL_BUILD)
	$(CXX) $(CXXFLAGS) -include $(BUILD)/build_id.h -c $< -o $@
$(PKG)/libmstab_b200_tl.so: $(TL_OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $^ -Xlinker -Bsymbolic -lcudart_static -ldl -lrt -lpthread

sass: $(CU_OBJS)
	for o in $(CU_OBJS); do $(CUDA_HOME)/bin/cuobjdump -sass $$o; done > $(BUILD)/kernels.sass

clean:
	rm -rf $(BUILD) $(PKG)/*.so

.PHONY: all product gen oracle ref clean sass timeline FORCE
FORCE:
