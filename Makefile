# Builds the C-ABI shared library for sm_100a (B200) in-tree.
NVCC      ?= /usr/local/cuda/bin/nvcc
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(EXTRA) -O3 -lineinfo -std=c++17 $(ARCH) -Xcompiler -fPIC -Xcompiler -Wall \
             -Xptxas -v --expt-relaxed-constexpr
PKG       := paper_2409_02912_b200
SRC_DIR   := $(PKG)/csrc
BUILD     ?= build
CU_SRCS   := $(wildcard $(SRC_DIR)/*.cu)
CPP_SRCS  := $(wildcard $(SRC_DIR)/*.cpp)
OBJS      := $(patsubst $(SRC_DIR)/%.cu,$(BUILD)/%.o,$(CU_SRCS)) $(patsubst $(SRC_DIR)/%.cpp,$(BUILD)/%.cpp.o,$(CPP_SRCS))
HDRS      := $(wildcard $(SRC_DIR)/*.h $(SRC_DIR)/*.cuh) include/nrx_b200.h
LIB       ?= $(PKG)/libnrx_b200.so

all: $(LIB)

$(BUILD)/%.o: $(SRC_DIR)/%.cu $(HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $@.ptxas.log || (cat $@.ptxas.log; false)

$(BUILD)/%.cpp.o: $(SRC_DIR)/%.cpp $(HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) -O3 -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall -c $< -o $@

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcuda

clean:
	rm -rf $(BUILD) $(LIB)

.PHONY: all clean
