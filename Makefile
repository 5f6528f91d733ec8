# Builds the B200-native engine (sm_100a only) and the test-only oracle libraries.
#
#   make            -> paper_2508_16508_b200/libabmx_cuda.so  + oracle/liboracle.so (+ oracle/_ref)
#   make cuda       -> only the product library
#
# -fmad=false: the reference's g++ x86-64 build never contracts a*b+c into an FMA, and the
# energy arithmetic (frac * E, E - child, E +/- gain) must round identically.

NVCC    ?= nvcc
ARCH    := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC -Xcompiler -Wall \
           -Xptxas -v
PKG     := paper_2508_16508_b200
SRC     := $(PKG)/csrc
OBJDIR  := build/obj
CU      := table predation ensemble agents traffic traffic_ens finance diag capi
OBJS    := $(addprefix $(OBJDIR)/,$(addsuffix .o,$(CU)))
HDRS    := $(wildcard $(SRC)/*.h $(SRC)/*.cuh) include/abmx_cuda.h

all: cuda oracle functor_cases

cuda: $(PKG)/libabmx_cuda.so

# test library: the header-only device functor API (include/abmx_cuda_functors.cuh) on the
# scenarios tests/test_functors_gpu.py compares with the reference (not part of the product)
functor_cases: build/libabmx_functor_cases.so

build/libabmx_functor_cases.so: tests/cpp/functor_cases.cu include/abmx_cuda_functors.cuh include/abmx_cuda.hpp \
		include/abmx_cuda.h $(PKG)/libabmx_cuda.so
	@mkdir -p build
	$(NVCC) $(ARCH) -O3 -std=c++17 -fmad=false -Xcompiler -fPIC -Iinclude -shared -o $@ $< \
		-L$(PKG) -labmx_cuda -Xlinker -rpath,'$$ORIGIN/../$(PKG)'

$(OBJDIR)/%.o: $(SRC)/%.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(OBJDIR)/$*.ptxas.txt || (cat $(OBJDIR)/$*.ptxas.txt; false)

$(PKG)/libabmx_cuda.so: $(OBJS)
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $(OBJS)

oracle: cuda
	$(MAKE) -C oracle all ref_cuda

clean:
	rm -rf build $(PKG)/libabmx_cuda.so
	$(MAKE) -C oracle clean

.PHONY: all cuda oracle functor_cases clean
