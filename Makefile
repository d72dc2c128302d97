# Top-level build: the sm_100a CUDA library (product) and the oracle (tests).
NVCC      ?= nvcc
PKG       := paper_2211_00224_b200
CSRC      := $(PKG)/csrc
LIB       := $(PKG)/libsolar_b200.so
CU_SRCS   := $(wildcard $(CSRC)/*.cu)
CU_OBJS   := $(patsubst $(CSRC)/%.cu,build/%.o,$(CU_SRCS))
NVFLAGS   := -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
             -Xcompiler -fPIC -Xcompiler -Wall -Iinclude --expt-relaxed-constexpr

.PHONY: all lib host oracle clean
all: lib host oracle
lib: $(LIB)

# C++ loadsched drop-in over the C ABI + its test driver
HOSTLIB   := $(PKG)/libloadsched_gpu.so
CUDA_HOME ?= /usr/local/cuda
host: $(HOSTLIB) tests/cpp/dropin_test
$(HOSTLIB): $(PKG)/host/loadsched_gpu.cpp include/loadsched_gpu.hpp include/lsg.h $(LIB)
	g++ -std=c++20 -O2 -fPIC -shared -Wall -Iinclude -I$(CUDA_HOME)/include $(PKG)/host/loadsched_gpu.cpp \
	    -L$(PKG) -lsolar_b200 -L$(CUDA_HOME)/lib64 -lcudart -Wl,-rpath,'$$ORIGIN' -o $@
tests/cpp/dropin_test: tests/cpp/dropin_test.cpp include/loadsched_gpu.hpp $(HOSTLIB)
	g++ -std=c++20 -O2 -Wall -Iinclude tests/cpp/dropin_test.cpp -L$(PKG) -lloadsched_gpu -lsolar_b200 \
	    -Wl,-rpath,'$$ORIGIN/../../$(PKG)' -o $@

build/%.o: $(CSRC)/%.cu $(wildcard $(CSRC)/*.cuh) include/lsg.h
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB): $(CU_OBJS)
	$(NVCC) -shared -cudart shared -gencode arch=compute_100a,code=sm_100a -o $@ $^

oracle:
	$(MAKE) -C oracle all

clean:
	rm -rf build $(LIB) $(HOSTLIB) tests/cpp/dropin_test
