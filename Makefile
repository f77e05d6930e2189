# Build everything in-tree (the .so files travel to the GPU box with gpurun).
#   make            -> oracle, generator, CUDA library
#   make oracle gen -> CPU-only parts
NVCC      ?= /usr/local/cuda/bin/nvcc
CXX       ?= g++
ARCH      := -gencode arch=compute_100a,code=sm_100a
# no fast-math and no FMA contraction: the path must be bit-reproducible
NVFLAGS   := -O3 -std=c++17 $(ARCH) -lineinfo -fmad=false -Xcompiler -fPIC \
             -Xptxas -v --expt-relaxed-constexpr
CXXFLAGS  := -O2 -std=c++17 -fPIC -ffp-contract=off -fno-fast-math -Wall

PKG       := paper_2003_04920_b200
CSRC      := $(PKG)/csrc
LIBPIRRT  := $(PKG)/lib/libpirrt.so
CU_SRCS   := $(wildcard $(CSRC)/*.cu)
CU_HDRS   := $(wildcard $(CSRC)/*.cuh) include/pirrt.h

all: oracle gen cuda

oracle: oracle/liboracle.so
gen: gen/libgen.so
cuda: $(LIBPIRRT)

oracle/liboracle.so: oracle/oracle.cpp oracle/oracle.h
	$(CXX) $(CXXFLAGS) -shared -o $@ oracle/oracle.cpp

gen/libgen.so: gen/rrg.cpp
	$(CXX) -O2 -std=c++17 -fPIC -pthread -Wall -shared -o $@ gen/rrg.cpp

$(LIBPIRRT): $(CU_SRCS) $(CU_HDRS)
	@mkdir -p $(PKG)/lib
	$(NVCC) $(NVFLAGS) -Iinclude -shared -o $@ $(CU_SRCS) -ldl 2> $(PKG)/lib/ptxas.log || (cat $(PKG)/lib/ptxas.log; exit 1)
	@grep -E "registers|spill" $(PKG)/lib/ptxas.log | sed 's/^/  /' | head -40

clean:
	rm -f oracle/liboracle.so gen/libgen.so $(LIBPIRRT)

.PHONY: all oracle gen cuda clean
