# Build of the B200 HEC triangular-solve library (sm_100a) and of the test
# oracles. `make` builds everything that can be built here:
#   paper_1606_00541_b200/libhecsolve_b200.so   product (C++ host setup + CUDA + C-ABI)
#   oracle/_build/libhecoracle.so                C restatement (tests / bench baseline only)
#   oracle/_ref/libhecref.so                     the reference itself (only if /root/reference exists)

CUDA_HOME ?= /usr/local/cuda
NVCC      := $(CUDA_HOME)/bin/nvcc -ccbin /usr/bin/g++
CXX       := /usr/bin/g++
ARCH      := -gencode arch=compute_100a,code=sm_100a

PKG   := paper_1606_00541_b200
SRC   := $(PKG)/csrc
OBJ   ?= build/obj
LIB   ?= $(PKG)/libhecsolve_b200.so

HOST_FLAGS := -O3 -std=c++20 -fPIC -fopenmp -ffp-contract=off -Wall -Wextra -Iinclude
CU_FLAGS   := -O3 -std=c++20 $(ARCH) -lineinfo -fmad=false -Xptxas -v $(EXTRA_CU_FLAGS) \
              -Xcompiler -fPIC,-fopenmp,-ffp-contract=off -Iinclude

HOST_SRCS := $(wildcard $(SRC)/host/*.cpp) $(wildcard $(SRC)/cuda/*.cpp)
CAPI_SRCS := $(wildcard $(SRC)/capi/*.cpp)
CU_SRCS   := $(wildcard $(SRC)/cuda/*.cu)

HOST_OBJS := $(patsubst $(SRC)/%.cpp,$(OBJ)/%.o,$(HOST_SRCS))
CAPI_OBJS := $(patsubst $(SRC)/%.cpp,$(OBJ)/%.o,$(CAPI_SRCS))
CU_OBJS   := $(patsubst $(SRC)/%.cu,$(OBJ)/%.cu.o,$(CU_SRCS))

HEADERS := $(wildcard include/*.h include/hecsolve/*.hpp $(SRC)/cuda/*.hpp $(SRC)/cuda/*.cuh)

BENCH_EXE := $(PKG)/bin/hecsolve_bench

.PHONY: all lib oracle clean
all: lib oracle

lib: $(LIB) $(BENCH_EXE)

# the reference's benchmark command line (tools/bench_main.cpp) over this library
$(BENCH_EXE): $(SRC)/tools/bench_main.cpp $(LIB) $(HEADERS)
	@mkdir -p $(dir $@)
	$(CXX) -O2 -std=c++20 -Iinclude -o $@ $< -L$(PKG) -lhecsolve_b200 -Wl,-rpath,'$$ORIGIN/..'

$(LIB): $(HOST_OBJS) $(CAPI_OBJS) $(CU_OBJS)
	$(NVCC) -shared $(ARCH) -cudart static -Xcompiler -fopenmp -o $@ $^ -lgomp -ldl

$(OBJ)/%.o: $(SRC)/%.cpp $(HEADERS)
	@mkdir -p $(dir $@)
	$(CXX) $(HOST_FLAGS) -I$(CUDA_HOME)/include -c $< -o $@

$(OBJ)/%.cu.o: $(SRC)/%.cu $(HEADERS)
	@mkdir -p $(dir $@)
	$(NVCC) $(CU_FLAGS) -c $< -o $@ 2> $@.ptxas.log || (cat $@.ptxas.log; exit 1)

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(LIB) $(BENCH_EXE)
	$(MAKE) -C oracle clean
