# Top-level build: the sm_100a CUDA library (product) and the oracle (tests).
NVCC      ?= nvcc
PKG       := paper_2211_00224_b200
CSRC      := $(PKG)/csrc
LIB       := $(PKG)/libsolar_b200.so
CU_SRCS   := $(wildcard $(CSRC)/*.cu)
CU_OBJS   := $(patsubst $(CSRC)/%.cu,build/%.o,$(CU_SRCS))
NVFLAGS   := -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
             -Xcompiler -fPIC -Xcompiler -Wall -Iinclude --expt-relaxed-constexpr

.PHONY: all lib oracle clean
all: lib oracle
lib: $(LIB)

build/%.o: $(CSRC)/%.cu $(CSRC)/common.cuh include/lsg.h
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB): $(CU_OBJS)
	$(NVCC) -shared -cudart shared -gencode arch=compute_100a,code=sm_100a -o $@ $^

oracle:
	$(MAKE) -C oracle all

clean:
	rm -rf build $(LIB)
