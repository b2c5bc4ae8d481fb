# Builds the sm_100a engine in-tree: paper_2407_20713_b200/lib/libsabr_b200.so
# (cross-compiles without a GPU).  `make oracle` builds the test-only checkers.

NVCC     ?= nvcc
HOSTCXX  := $(shell test -x /usr/bin/g++ && echo /usr/bin/g++ || echo g++)
ARCH     := -gencode arch=compute_100a,code=sm_100a
NVFLAGS  := $(ARCH) -O3 -lineinfo -std=c++17 -ccbin $(HOSTCXX) -Iinclude \
            -Xcompiler -fPIC,-fvisibility=hidden,-O3 -Xptxas -O3 --expt-relaxed-constexpr
SRC_DIR  := paper_2407_20713_b200/csrc
OBJ_DIR  := build/obj
LIB      := paper_2407_20713_b200/lib/libsabr_b200.so

CU_SRCS  := $(SRC_DIR)/kernels_sa.cu $(SRC_DIR)/kernels_mc.cu $(SRC_DIR)/engine.cu \
            $(SRC_DIR)/t2_driver.cu $(SRC_DIR)/peak.cu $(SRC_DIR)/kernels_c2f.cu $(SRC_DIR)/kernels_bs.cu
CPP_SRCS := $(SRC_DIR)/xoshiro_jump.cpp
# host-only C++ (binary128 arithmetic, which nvcc's front end does not take)
HOST_SRCS := $(SRC_DIR)/slice_qr.cpp
OBJS     := $(patsubst $(SRC_DIR)/%.cu,$(OBJ_DIR)/%.o,$(CU_SRCS)) \
            $(patsubst $(SRC_DIR)/%.cpp,$(OBJ_DIR)/%.o,$(CPP_SRCS)) \
            $(patsubst $(SRC_DIR)/%.cpp,$(OBJ_DIR)/host_%.o,$(HOST_SRCS))
HDRS     := $(wildcard $(SRC_DIR)/*.hpp $(SRC_DIR)/*.cuh) include/sabr_b200.h

.PHONY: all lib oracle clean

all: lib

lib: $(LIB)

$(OBJ_DIR)/%.o: $(SRC_DIR)/%.cu $(HDRS)
	@mkdir -p $(OBJ_DIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(OBJ_DIR)/%.o: $(SRC_DIR)/%.cpp $(HDRS)
	@mkdir -p $(OBJ_DIR)
	$(NVCC) $(NVFLAGS) -x cu -c $< -o $@

$(OBJ_DIR)/host_%.o: $(SRC_DIR)/%.cpp $(HDRS)
	@mkdir -p $(OBJ_DIR)
	$(HOSTCXX) -std=c++17 -O2 -fPIC -fvisibility=hidden -c $< -o $@

$(LIB): $(OBJS)
	@mkdir -p $(dir $(LIB))
	$(NVCC) $(ARCH) -shared -ccbin $(HOSTCXX) -o $@ $(OBJS) -ldl

oracle:
	$(MAKE) -C oracle all

clean:
	rm -rf build $(LIB)
