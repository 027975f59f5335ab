# Builds the product (sm_100a CUDA + C ABI + C++ drop-in library), the C++
# parity tests, and the CPU oracle (test infrastructure, oracle/Makefile).
NVCC      ?= nvcc
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := -O3 -lineinfo -std=c++17 $(ARCH) -Xcompiler -fPIC -Iinclude -Ipaper_2603_21444_b200/csrc \
             --expt-relaxed-constexpr -Xptxas -warn-spills
CXXFLAGS  := -O3 -std=c++20 -fPIC -Iinclude -Wall -Wextra
PKG       := paper_2603_21444_b200
LIBDIR    := $(PKG)/lib
OBJDIR    := build/obj
CU_SRCS   := $(wildcard $(PKG)/csrc/*.cu)
CU_OBJS   := $(patsubst $(PKG)/csrc/%.cu,$(OBJDIR)/%.o,$(CU_SRCS))
HOST_SRCS := $(wildcard $(PKG)/host/*.cpp)
HOST_OBJS := $(patsubst $(PKG)/host/%.cpp,$(OBJDIR)/host_%.o,$(HOST_SRCS))
CAPI_LIB  := $(LIBDIR)/libspgb200.so
CXX_LIB   := $(LIBDIR)/libspgsim_b200.so
CUDA_LIB  := /usr/local/cuda/lib64

all: $(CAPI_LIB) $(CXX_LIB) tests/cpp/test_csr_b200 oracle

$(OBJDIR)/%.o: $(PKG)/csrc/%.cu $(wildcard $(PKG)/csrc/*.cuh) include/spg/capi.h
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(CAPI_LIB): $(CU_OBJS)
	@mkdir -p $(LIBDIR)
	$(NVCC) $(ARCH) -shared -o $@ $(CU_OBJS) -cudart static

$(OBJDIR)/host_%.o: $(PKG)/host/%.cpp $(wildcard include/spgsim/*.hpp) include/spg/capi.h
	@mkdir -p $(OBJDIR)
	g++ $(CXXFLAGS) -c $< -o $@

$(CXX_LIB): $(HOST_OBJS) $(CAPI_LIB)
	g++ -shared -o $@ $(HOST_OBJS) -L$(LIBDIR) -lspgb200 -Wl,-rpath,'$$ORIGIN'

tests/cpp/test_csr_b200: tests/cpp/test_csr_b200.cpp tests/cpp/mini_test.hpp $(CXX_LIB)
	g++ $(CXXFLAGS) -o $@ $< -L$(LIBDIR) -lspgsim_b200 -lspgb200 -Wl,-rpath,'$$ORIGIN/../../$(LIBDIR)'

oracle:
	$(MAKE) -C oracle lib/libspgoracle.so
	@if [ -d /root/reference/proj ]; then $(MAKE) -C oracle ref; fi

clean:
	rm -rf build $(LIBDIR) tests/cpp/test_csr_b200

.PHONY: all oracle clean
