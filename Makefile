# Product build: sm_100a CUDA apply library (and the host descriptor library).
# Outputs land in-tree under paper_2310_16668_b200/lib/ so they travel to the
# GPU box with the repo snapshot.  `make oracle` builds the test-only checkers
# (oracle/Makefile).
NVCC     ?= /usr/local/cuda/bin/nvcc
CXX      := g++
PKG      := paper_2310_16668_b200
SRC      := $(PKG)/csrc
LIB      := $(PKG)/lib
OBJ      := build/obj
ARCH     := -gencode arch=compute_100a,code=sm_100a
NVFLAGS  := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude -I$(SRC) \
            --expt-relaxed-constexpr -Xptxas -v -Xcompiler -fopenmp
CXXFLAGS := -std=c++17 -O2 -fopenmp -fPIC -Iinclude -I$(SRC) -I/usr/local/cuda/include

GPU_CU   := $(SRC)/kernels_translate.cu $(SRC)/kernels_tree.cu $(SRC)/kernels_multi.cu $(SRC)/skel_gpu.cu \
            $(SRC)/tree_gpu.cu $(SRC)/sfmm_gpu.cu $(SRC)/sfmm_multi.cu
GPU_OBJS := $(patsubst $(SRC)/%.cu,$(OBJ)/%.o,$(GPU_CU)) $(OBJ)/plan_build.o
HDRS     := include/sfmm_gpu.h $(SRC)/plan.h $(SRC)/common.cuh $(SRC)/launch.h $(SRC)/plan_build.h $(SRC)/fastmath.cuh $(SRC)/log_table.inc

.PHONY: all gpu host probe oracle clean
all: gpu host probe check-bin

HOST_SRC  := $(SRC)/host
HOST_CPP  := $(HOST_SRC)/host_api.cpp
HOST_OBJS := $(patsubst $(HOST_SRC)/%.cpp,$(OBJ)/host_%.o,$(HOST_CPP))
HOSTFLAGS := -std=c++17 -O3 -march=x86-64-v3 -fopenmp -fPIC -Iinclude -I$(HOST_SRC) \
             -fno-math-errno -fcx-limited-range -ffp-contract=off

host: $(LIB)/libsfmm_host.so

$(OBJ)/host_%.o: $(HOST_SRC)/%.cpp $(HOST_SRC)/host.h include/sfmm_host.h include/sfmm_gpu.h
	@mkdir -p $(OBJ)
	$(CXX) $(HOSTFLAGS) -c $< -o $@

$(LIB)/libsfmm_host.so: $(HOST_OBJS)
	@mkdir -p $(LIB)
	$(CXX) -shared -fopenmp $^ -o $@

gpu: $(LIB)/libsfmm_gpu.so

$(OBJ)/%.o: $(SRC)/%.cu $(HDRS)
	@mkdir -p $(OBJ)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(OBJ)/$*.ptxas.txt || (cat $(OBJ)/$*.ptxas.txt; false)

$(OBJ)/plan_build.o: $(SRC)/plan_build.cpp $(HDRS)
	@mkdir -p $(OBJ)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(LIB)/libsfmm_gpu.so: $(GPU_OBJS)
	@mkdir -p $(LIB)
	$(NVCC) $(ARCH) -shared -o $@ $^ -lcudart_static -lgomp -lpthread -ldl -lrt

# measurement / test hooks (include/sfmm_probe.h): not part of the apply ABI
probe: $(LIB)/libsfmm_probe.so

$(LIB)/libsfmm_probe.so: $(SRC)/probe/sfmm_probe.cu include/sfmm_probe.h $(SRC)/fastmath.cuh $(SRC)/log_table.inc
	@mkdir -p $(LIB) $(OBJ)
	$(NVCC) $(NVFLAGS) -shared -o $@ $< -lcudart_static -ldl -lrt -lpthread 2> $(OBJ)/probe.ptxas.txt || (cat $(OBJ)/probe.ptxas.txt; false)

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(LIB)

# C++ check of the distributed precompute header (run by tests/test_distributed_precompute.py)
check-bin: build/bin/dist_precompute_check

build/bin/dist_precompute_check: tests/cpp/dist_precompute_check.cpp include/sfmm_gpu_dist.hpp include/sfmm_gpu.h $(LIB)/libsfmm_gpu.so
	@mkdir -p build/bin
	$(CXX) -std=c++17 -O2 -Iinclude $< -L$(LIB) -lsfmm_gpu -Wl,-rpath,'$$ORIGIN/../../$(LIB)' -o $@
