# Builds the in-tree C-ABI library (sm_100a) and the oracle's C helpers.
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
CXXFLAGS := -O3 -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall -lineinfo
# `make TRACE=1` (after touching csrc/tc.cu) compiles the GEMM event log in (SYNO_TC_TRACE=<file>)
ifdef TRACE
CXXFLAGS += -DSYNO_TC_TRACE_EVENTS
endif
# `make SUSPEND=1` (after touching csrc/tc.cu): every GEMM barrier wait uses the suspending try_wait
ifdef SUSPEND
CXXFLAGS += -DSYNO_MBAR_SUSPEND
endif
# `make DBG=1` (after touching csrc/tc.cu) compiles the SYNO_TC_DEBUG switches in
ifdef DBG
CXXFLAGS += -DSYNO_TC_DBG_SWITCHES
endif
PKG := paper_2410_23745_b200
SRC := $(PKG)/csrc
OBJ := build/obj
HOST_SRCS := symbolic graph nest plan simplify shapedist capi
CUDA_SRCS := engine tc
OBJS := $(addprefix $(OBJ)/,$(addsuffix .o,$(HOST_SRCS) $(CUDA_SRCS)))
HDRS := $(wildcard $(SRC)/*.hpp) $(wildcard $(SRC)/*.cuh) include/syno.h

all: $(PKG)/libsyno.so

$(OBJ)/%.o: $(SRC)/%.cpp $(HDRS)
	@mkdir -p $(OBJ)
	$(NVCC) $(ARCH) $(CXXFLAGS) -x cu -c $< -o $@

$(OBJ)/%.o: $(SRC)/%.cu $(HDRS)
	@mkdir -p $(OBJ)
	$(NVCC) $(ARCH) $(CXXFLAGS) -Xptxas -v -c $< -o $@ 2> $(OBJ)/$*.ptxas.txt || (cat $(OBJ)/$*.ptxas.txt; false)

$(PKG)/libsyno.so: $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcudart -lcuda

clean:
	rm -rf build $(PKG)/libsyno.so

.PHONY: all clean
