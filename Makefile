# Build of the B200-native FastH library (sm_100a) and the test oracle.
#
#   make            -> paper_2009_13977_b200/lib/libfasth_b200.so + oracle
#   make lib        -> the product library only
#   make oracle     -> oracle/_build/liboracle.so (+ oracle/_ref when the
#                      reference tree is present)
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -O3 \
           -Iinclude -Ipaper_2009_13977_b200/csrc --expt-relaxed-constexpr
SRC_DIR := paper_2009_13977_b200/csrc
OBJ_DIR := build/obj
LIB := paper_2009_13977_b200/lib/libfasth_b200.so
CU_SRCS := $(wildcard $(SRC_DIR)/*.cu)
CPP_SRCS := $(wildcard $(SRC_DIR)/*.cpp)
OBJS := $(patsubst $(SRC_DIR)/%.cu,$(OBJ_DIR)/%.o,$(CU_SRCS)) \
        $(patsubst $(SRC_DIR)/%.cpp,$(OBJ_DIR)/%.o,$(CPP_SRCS))
HDRS := $(wildcard $(SRC_DIR)/*.h $(SRC_DIR)/*.cuh) include/fasth_b200.h

all: lib oracle

lib: $(LIB)

$(OBJ_DIR)/%.o: $(SRC_DIR)/%.cu $(HDRS)
	@mkdir -p $(OBJ_DIR)
	$(NVCC) $(NVFLAGS) -Xptxas -v -c $< -o $@ 2> $(OBJ_DIR)/$*.ptxas.txt || (cat $(OBJ_DIR)/$*.ptxas.txt; false)

$(OBJ_DIR)/%.o: $(SRC_DIR)/%.cpp $(HDRS)
	@mkdir -p $(OBJ_DIR)
	$(NVCC) $(NVFLAGS) -x cu -c $< -o $@

$(LIB): $(OBJS)
	@mkdir -p $(dir $(LIB))
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -cudart static

oracle:
	$(MAKE) -s -C oracle

clean:
	rm -rf build $(LIB)

.PHONY: all lib oracle clean
