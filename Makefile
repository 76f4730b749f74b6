# Build of the B200-native matrix-free PCG (in-tree; the .so files travel to
# the GPU box with the gpurun snapshot).
#
#   paper_1302_7193_b200/libacg_cuda.so      sm_100a kernels + C ABI (include/acg.h)
#   paper_1302_7193_b200/_anisocg*.so        host C++ shim (namespace anisocg) + pybind11
#   oracle/liboracle.so, oracle/_ref/*       CPU checkers (oracle/Makefile)
PY      ?= python3
NVCC    ?= nvcc
PKG     := paper_1302_7193_b200
CSRC    := $(PKG)/csrc
EXT     := $(shell $(PY) -c 'import sysconfig;print(sysconfig.get_config_var("EXT_SUFFIX"))')
PYINC   := $(shell $(PY) -c 'import sysconfig;print(sysconfig.get_paths()["include"])')
PBINC   := $(shell $(PY) -c 'import pybind11;print(pybind11.get_include())')
CUDA    ?= /usr/local/cuda
ARCH    := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -lineinfo -O3 -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall
CXXFLAGS:= -O2 -std=c++20 -fPIC -Wall -ffp-contract=off -Iinclude -I$(CUDA)/include

LIB     := $(PKG)/libacg_cuda.so
PYMOD   := $(PKG)/_anisocg$(EXT)
HOSTSRC := $(CSRC)/host/grid.cpp $(CSRC)/host/profile.cpp $(CSRC)/host/shim.cpp \
           $(CSRC)/host/cost_model.cpp $(CSRC)/host/io.cpp
HDRS    := include/acg.h $(wildcard include/anisocg/*.hpp) $(CSRC)/acg_internal.h

.PHONY: all lib py oracle micro clean
all: lib py oracle micro

# sanitizer evidence kernel (tests/test_sanitizers.py)
micro: scripts/micro/tmem_synccheck
scripts/micro/tmem_synccheck: scripts/micro/tmem_synccheck.cu
	$(NVCC) $(ARCH) -o $@ $<

lib: $(LIB)
py: $(PYMOD)

build/acg_kernels.o: $(CSRC)/acg_kernels.cu $(CSRC)/acg_internal.h $(wildcard $(CSRC)/*.cuh)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -Xptxas -v -c $< -o $@ 2> build/ptxas_kernels.log || (cat build/ptxas_kernels.log; false)

build/acg_runtime.o: $(CSRC)/acg_runtime.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB): build/acg_kernels.o build/acg_runtime.o
	$(NVCC) $(ARCH) -shared -o $@ $^ -cudart static -ldl -lpthread

$(PYMOD): $(CSRC)/python/bindings.cpp $(HOSTSRC) $(HDRS) $(LIB)
	g++ $(CXXFLAGS) -shared -I$(PYINC) -I$(PBINC) -o $@ $(CSRC)/python/bindings.cpp $(HOSTSRC) \
	    -L$(PKG) -lacg_cuda -Wl,-rpath,'$$ORIGIN'

oracle: lib
	$(MAKE) -C oracle PY=$(PY)

clean:
	rm -rf build $(LIB) $(PYMOD)
