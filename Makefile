# Product build: sm_100a CUDA apply library (and the host precompute library).
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
            --expt-relaxed-constexpr -Xptxas -v
CXXFLAGS := -std=c++17 -O2 -fPIC -Iinclude -I$(SRC) -I/usr/local/cuda/include

GPU_CU   := $(SRC)/kernels_translate.cu $(SRC)/kernels_tree.cu $(SRC)/sfmm_gpu.cu
GPU_OBJS := $(patsubst $(SRC)/%.cu,$(OBJ)/%.o,$(GPU_CU)) $(OBJ)/plan_build.o
HDRS     := include/sfmm_gpu.h $(SRC)/common.cuh $(SRC)/launch.h $(SRC)/plan_build.h

.PHONY: all gpu oracle clean
all: gpu

gpu: $(LIB)/libsfmm_gpu.so

$(OBJ)/%.o: $(SRC)/%.cu $(HDRS)
	@mkdir -p $(OBJ)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(OBJ)/$*.ptxas.txt || (cat $(OBJ)/$*.ptxas.txt; false)

$(OBJ)/plan_build.o: $(SRC)/plan_build.cpp $(HDRS)
	@mkdir -p $(OBJ)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(LIB)/libsfmm_gpu.so: $(GPU_OBJS)
	@mkdir -p $(LIB)
	$(NVCC) $(ARCH) -shared -o $@ $^ -lcudart_static -lpthread -ldl -lrt

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(LIB)
