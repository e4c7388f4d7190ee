# Builds the engine's shared library in-tree (it travels to the GPU box with
# gpurun) and the oracle checkers.
#   paper_2108_03076_b200/libcltk_b200.so  -- sm_100a kernels + C++ host + C-ABI
NVCC     ?= /usr/local/cuda/bin/nvcc
HOSTCXX  := /usr/bin/g++
NLOHMANN ?= /opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty
PKG      := paper_2108_03076_b200
SRC      := $(PKG)/csrc
OBJ      := build/obj
LIB      := $(PKG)/libcltk_b200.so
ARCH     := -gencode arch=compute_100a,code=sm_100a

# EXTRA_DEFS: experiment builds (e.g. make lib OBJ=build/obj_x LIB=build/variants/x/libcltk_b200.so
# EXTRA_DEFS=-DCLTK_BLOCK=64); the product build leaves it empty
EXTRA_DEFS ?=
CXXFLAGS := $(EXTRA_DEFS) -std=c++17 -O2 -fPIC -ffp-contract=off -Wall -Wno-unused-function \
            -I$(NLOHMANN) -I/usr/local/cuda/include -Iinclude
NVFLAGS  := $(EXTRA_DEFS) $(ARCH) -std=c++17 -O3 -lineinfo -fmad=false -ccbin $(HOSTCXX) \
            -Xcompiler -fPIC -Xptxas -v -Iinclude

HOST_SRCS := host_model compiler engine capi sobol_table jit reindex nccl_comm
HOST_OBJS := $(addprefix $(OBJ)/,$(addsuffix .o,$(HOST_SRCS))) $(OBJ)/jit_sources.o
# device headers embedded for the NVRTC build (csrc/jit.cpp)
JIT_HDRS  := $(SRC)/engine_device.cuh $(SRC)/engine_types.h $(SRC)/program.h \
             $(SRC)/glibc_math.h $(SRC)/glibc_tables.h
CU_OBJS   := $(OBJ)/mc_engine.o $(OBJ)/mc_engine_qmc.o $(OBJ)/mc_engine_fault.o
HDRS      := $(wildcard $(SRC)/*.hpp $(SRC)/*.h $(SRC)/*.cuh) include/cltk_b200.h

.PHONY: all lib oracle testlib clean
all: lib oracle testlib

lib: $(LIB)

$(OBJ)/%.o: $(SRC)/%.cpp $(HDRS)
	@mkdir -p $(OBJ)
	$(HOSTCXX) $(CXXFLAGS) -c $< -o $@

$(OBJ)/jit_sources.cpp: $(JIT_HDRS) tools/embed_sources.py
	@mkdir -p $(OBJ)
	python3 tools/embed_sources.py $@ $(JIT_HDRS)

$(OBJ)/jit_sources.o: $(OBJ)/jit_sources.cpp
	$(HOSTCXX) $(CXXFLAGS) -c $< -o $@

# three translation units compiled in parallel (mc_engine.cu CLTK_AOT_PART)
$(CU_OBJS): $(OBJ)/%.o: $(SRC)/%.cu $(SRC)/mc_engine.cu $(HDRS)
	@mkdir -p $(OBJ)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(OBJ)/$*.ptxas.txt || (cat $(OBJ)/$*.ptxas.txt; false)
	@grep -E "Used|spill" $(OBJ)/$*.ptxas.txt | head -40

$(LIB): $(HOST_OBJS) $(CU_OBJS)
	$(NVCC) $(ARCH) -shared -ccbin $(HOSTCXX) -cudart static -o $@ $^ -ldl

oracle:
	$(MAKE) -C oracle all

clean:
	rm -rf build $(LIB)

# test helper: host build of csrc/glibc_math.h (checked against the system libm)
testlib: build/libgm_check.so
build/libgm_check.so: tests/native/gm_check.cpp $(SRC)/glibc_math.h $(SRC)/glibc_tables.h
	@mkdir -p build
	$(HOSTCXX) -std=c++17 -O2 -fPIC -shared -ffp-contract=off -o $@ $< -lm
