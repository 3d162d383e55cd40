# Build for the B200-native SI framework.
#   make            planner library + CUDA library (sm_100a) + CPU oracle
#   make planner    libweft_b200.so   (host C++ planner, drop-in weft API, JSON C ABI)
#   make cuda       libdh_b200.so     (sm_100a kernels, runtime, executor, dh_* C ABI)
#   make oracle     oracle/_ref/* and oracle/liblayer_oracle (see oracle/Makefile)
# Outputs land in-tree (paper_2411_15871_b200/lib/) so they travel to the GPU box.

CXX      ?= g++
LINK_CXX ?= /usr/bin/g++
NVCC     ?= /usr/local/cuda/bin/nvcc
PKG      := paper_2411_15871_b200
LIB      := $(PKG)/lib
OBJ      := build
JOBS     ?= 8

CXXFLAGS := -std=c++20 -O2 -fPIC -ffp-contract=off -Wall -Wextra -Wno-unused-parameter \
            -Iinclude -Ithird_party
ARCH     := -gencode arch=compute_100a,code=sm_100a
NVFLAGS  := -std=c++20 -O3 $(ARCH) -cudart shared -lineinfo -Xcompiler -fPIC -Xcompiler -ffp-contract=off \
            -Iinclude -Ithird_party -I$(PKG)/csrc/cuda --expt-relaxed-constexpr \
            -Xptxas -warn-spills

PLANNER_SRC := $(wildcard $(PKG)/csrc/planner/*.cpp)
PLANNER_OBJ := $(patsubst $(PKG)/csrc/planner/%.cpp,$(OBJ)/planner/%.o,$(PLANNER_SRC))
CUDA_SRC    := $(wildcard $(PKG)/csrc/cuda/*.cu)
CUDA_OBJ    := $(patsubst $(PKG)/csrc/cuda/%.cu,$(OBJ)/cuda/%.o,$(CUDA_SRC))
RT_SRC      := $(wildcard $(PKG)/csrc/runtime/*.cpp)
RT_OBJ      := $(patsubst $(PKG)/csrc/runtime/%.cpp,$(OBJ)/runtime/%.o,$(RT_SRC))
CUDA_HDR    := $(wildcard $(PKG)/csrc/cuda/*.cuh) $(wildcard include/*.h)

.PHONY: all planner cuda oracle clean
all: planner cuda oracle

planner: $(LIB)/libweft_b200.so
cuda: $(LIB)/libdh_b200.so
oracle: planner
	$(MAKE) -C oracle

$(OBJ)/planner/%.o: $(PKG)/csrc/planner/%.cpp $(wildcard include/weft/*.hpp) $(PKG)/csrc/planner/lane_sim.hpp
	@mkdir -p $(dir $@)
	$(CXX) $(CXXFLAGS) -c $< -o $@

# Linked by the system g++ so that libstdc++ is the shared system copy: a
# toolchain that only offers a static libstdc++ would export a private copy
# that clashes with the one numpy/torch load into the same process.
$(LIB)/libweft_b200.so: $(PLANNER_OBJ)
	@mkdir -p $(LIB)
	$(LINK_CXX) -shared -o $@ $^ -pthread

$(OBJ)/cuda/%.o: $(PKG)/csrc/cuda/%.cu $(CUDA_HDR)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) $(NVFLAGS_EXTRA) -c $< -o $@

$(OBJ)/runtime/%.o: $(PKG)/csrc/runtime/%.cpp $(CUDA_HDR) $(wildcard include/weft/*.hpp) \
                    $(wildcard $(PKG)/csrc/runtime/*.hpp) $(PKG)/csrc/planner/lane_sim.hpp
	@mkdir -p $(dir $@)
	$(CXX) $(CXXFLAGS) -I/usr/local/cuda/include -I$(PKG)/csrc/planner -c $< -o $@

$(LIB)/libdh_b200.so: $(CUDA_OBJ) $(RT_OBJ) $(PLANNER_OBJ)
	@mkdir -p $(LIB)
	$(NVCC) -shared -cudart shared $(ARCH) -o $@ $^ -L/usr/local/cuda/lib64 -lcuda -lnccl -Xlinker -rpath,/usr/local/cuda/lib64

clean:
	rm -rf $(OBJ) $(LIB)
	$(MAKE) -C oracle clean
