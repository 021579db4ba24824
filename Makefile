# Builds the sm_100a kernel layer + C++ host engine into one in-tree shared
# library (paper_2110_03888_b200/libp2r.so) and the reference oracle.
NVCC    ?= nvcc
CXX     ?= g++
ARCH    := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall \
           -Iinclude -Ipaper_2110_03888_b200/csrc --expt-relaxed-constexpr
PKG     := paper_2110_03888_b200
CSRC    := $(PKG)/csrc
BUILD   := build
CU_SRCS := $(wildcard $(CSRC)/*.cu)
CPP_SRCS:= $(wildcard $(CSRC)/engine/*.cpp)
CU_OBJS := $(patsubst $(CSRC)/%.cu,$(BUILD)/%.o,$(CU_SRCS))
CPP_OBJS:= $(patsubst $(CSRC)/engine/%.cpp,$(BUILD)/engine/%.o,$(CPP_SRCS))
LIB     := $(PKG)/libp2r.so

DROPIN  := $(BUILD)/dropin_mini_controller
# diagnostic build (A/B variants selected by env: legacy mma.sync attention, one-tile
# attention backward at hd 64, bulk-ring LayerNorm forward, plain gate kernel); the
# product library does not carry them. Loaded through P2R_LIB by tests / scripts.
DIAG_SRCS := attention attention_bwd_tc moe norm_embed_ce
DIAG_OBJS := $(patsubst %,$(BUILD)/diag/%.o,$(DIAG_SRCS))
DIAG_LIB  := $(BUILD)/libp2r_diag.so

all: $(LIB) $(DROPIN) $(DIAG_LIB)

$(BUILD)/diag/%.o: $(CSRC)/%.cu $(wildcard $(CSRC)/*.cuh) $(wildcard $(CSRC)/*.h) include/p2r_cuda.h
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -DP2R_DIAG -c $< -o $@

$(DIAG_LIB): $(DIAG_OBJS) $(filter-out $(patsubst %,$(BUILD)/%.o,$(DIAG_SRCS)),$(CU_OBJS)) $(CPP_OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $^ -cudart static

# a reference-style controller compiled against the drop-in headers, linked with libp2r.so
$(DROPIN): tests/dropin/mini_controller.cpp $(LIB) $(wildcard include/p2r/*.hpp)
	@mkdir -p $(dir $@)
	$(CXX) -std=c++20 -O2 -Wall -Iinclude -o $@ $< -L$(PKG) -l:libp2r.so -Wl,-rpath,'$$ORIGIN/../$(PKG)'

$(BUILD)/%.o: $(CSRC)/%.cu $(wildcard $(CSRC)/*.cuh) $(wildcard $(CSRC)/*.h) include/p2r_cuda.h
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(BUILD)/engine/%.o: $(CSRC)/engine/%.cpp $(wildcard $(CSRC)/engine/*.hpp) $(wildcard include/p2r/*.hpp) $(wildcard include/*.h)
	@mkdir -p $(dir $@)
	$(CXX) -std=c++20 -O2 -fPIC -Wall -Iinclude -I/usr/local/cuda/include -c $< -o $@

$(LIB): $(CU_OBJS) $(CPP_OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $^ -cudart static

oracle:
	bash oracle/build_ref.sh

clean:
	rm -rf $(BUILD) $(LIB)

.PHONY: all clean oracle
