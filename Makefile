# Build of the B200 (sm_100a) library and the oracle checker.
#   make            -> paper_1606_01216_b200/lib/libmgpu.so  (+ oracle/liboracle.so)
#   make ref        -> oracle/_ref/libmorref.so  (needs /root/reference; checker only)
NVCC    ?= nvcc
CXX     ?= g++
ARCH    := -gencode arch=compute_100a,code=sm_100a
PKG     := paper_1606_01216_b200
SRC     := $(PKG)/csrc
LIBDIR  := $(PKG)/lib
OBJDIR  := build/obj
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude -I$(SRC) -Xptxas -v
CXXFLAGS:= -O2 -std=c++17 -fPIC -Iinclude -Wall -Wextra

CU_SRCS  := $(wildcard $(SRC)/*.cu)
CPP_SRCS := $(wildcard $(SRC)/*.cpp)
CU_OBJS  := $(patsubst $(SRC)/%.cu,$(OBJDIR)/%.o,$(CU_SRCS))
CPP_OBJS := $(patsubst $(SRC)/%.cpp,$(OBJDIR)/%.cpp.o,$(CPP_SRCS))

REFINC  ?= /root/reference/proj/include

.PHONY: all lib shim oracle ref parity clean

all: lib oracle

lib: $(LIBDIR)/libmgpu.so

$(OBJDIR) $(LIBDIR):
	mkdir -p $@

$(OBJDIR)/cg.o $(OBJDIR)/cg_stream.o: $(SRC)/cg_common.cuh

$(OBJDIR)/%.o: $(SRC)/%.cu $(SRC)/internal.cuh include/mgpu.h | $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $@.ptxas.log || (cat $@.ptxas.log; exit 1)

$(OBJDIR)/%.cpp.o: $(SRC)/%.cpp include/mgpu.h | $(OBJDIR)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(LIBDIR)/libmgpu.so: $(CU_OBJS) $(CPP_OBJS) | $(LIBDIR)
	$(NVCC) $(ARCH) -shared -o $@ $^ -lcudart -ldl

# C++ drop-in backend: compiled against the reference's own headers (only
# where /root/reference exists); the .so travels to the GPU box.
shim: $(LIBDIR)/libmor_cuda.so

$(LIBDIR)/libmor_cuda.so: $(PKG)/host/cuda_backend.cpp $(PKG)/host/capi.cpp $(PKG)/host/cuda_backend.hpp include/mor_cuda.h $(LIBDIR)/libmgpu.so
	$(CXX) -std=c++20 -O2 -fPIC -shared -Wall -Wextra -I$(REFINC) -Iinclude -I$(PKG)/host -o $@ \
	  $(PKG)/host/cuda_backend.cpp $(PKG)/host/capi.cpp -L$(LIBDIR) -lmgpu -Wl,-rpath,'$$ORIGIN'

# Parity driver: reference CgBackend vs CudaCgBackend (checker, lives in oracle/_ref)
parity: shim ref
	$(CXX) -std=c++20 -O2 -Wall -I$(REFINC) -Iinclude -I$(PKG)/host -include functional -o oracle/_ref/backend_parity \
	  tests/cpp/backend_parity.cpp $(filter-out oracle/_ref/ref_shim.o,$(wildcard oracle/_ref/*.o)) \
	  -L$(LIBDIR) -lmor_cuda -lmgpu -Wl,-rpath,'$$ORIGIN/../../$(LIBDIR)' -lpthread

oracle:
	$(MAKE) -C oracle oracle

ref:
	$(MAKE) -C oracle ref

clean:
	rm -rf build $(LIBDIR)
	$(MAKE) -C oracle clean

# Experiment build (tools/fma_experiment.py): cg_cluster_v2 with DFMA terms.  Not the product.
fma-exp: $(LIBDIR)/exp/libmgpu_fma.so

$(OBJDIR)/fma/cg_cluster.o: $(SRC)/cg_cluster.cu $(SRC)/internal.cuh include/mgpu.h
	mkdir -p $(OBJDIR)/fma
	$(NVCC) $(NVFLAGS) -DMGPU_CLUSTER_FMA -c $< -o $@ 2> $@.ptxas.log || (cat $@.ptxas.log; exit 1)

$(LIBDIR)/exp/libmgpu_fma.so: $(filter-out $(OBJDIR)/cg_cluster.o,$(CU_OBJS)) $(OBJDIR)/fma/cg_cluster.o $(CPP_OBJS)
	mkdir -p $(LIBDIR)/exp
	$(NVCC) $(ARCH) -shared -o $@ $^ -lcudart -ldl
