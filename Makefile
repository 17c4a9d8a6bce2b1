# Build every native artefact in-tree (the .so files travel to the GPU box
# with the gpurun snapshot; they are git-ignored).
#
#   kurgen/libkurgen.so                 seeded input generator (shared inputs only)
#   oracle/liboracle.so                 CPU oracle — TEST INFRASTRUCTURE ONLY
#   paper_2102_07167_b200/libkur.so     the product: C-ABI + host builder + sm_100a kernels

NVCC      := /usr/local/cuda/bin/nvcc -ccbin /usr/bin/g++
CXX       := /usr/bin/g++
CC        := /usr/bin/gcc
ARCH      := -gencode arch=compute_100a,code=sm_100a
PYSITE    := $(shell python -c "import sysconfig;print(sysconfig.get_paths()['purelib'])")
NCCL_INC  := $(PYSITE)/nvidia/nccl/include
NCCL_LIB  := $(PYSITE)/nvidia/nccl/lib

PKG       := paper_2102_07167_b200
KUR_SRCS  := $(PKG)/csrc/builder.cpp $(PKG)/csrc/api.cpp $(PKG)/csrc/kernels.cu
KUR_HDRS  := include/kur.h $(PKG)/csrc/plan.h $(PKG)/csrc/kernels.h

all: kurgen/libkurgen.so oracle/liboracle.so $(PKG)/libkur.so

kurgen/libkurgen.so: kurgen/kurgen.cpp
	$(CXX) -O2 -std=c++17 -fopenmp -fPIC -shared -o $@ $<

# The oracle is plain C99, fp64, no fast-math, no FMA contraction.
oracle/liboracle.so: oracle/kur_oracle.c
	$(CC) -O2 -std=c99 -fno-fast-math -ffp-contract=off -fopenmp -fPIC -shared -o $@ $< -lm

$(PKG)/libkur.so: $(KUR_SRCS) $(KUR_HDRS)
	$(NVCC) $(ARCH) -O3 -lineinfo -std=c++17 -Iinclude -I$(NCCL_INC) \
	  -Xcompiler -fPIC,-fopenmp,-O3 -Xptxas -v -shared -o $@ $(KUR_SRCS) \
	  -L$(NCCL_LIB) -l:libnccl.so.2 -Xlinker -rpath,$(NCCL_LIB) -lgomp 2> $(PKG)/ptxas.log || \
	  (cat $(PKG)/ptxas.log; exit 1)

# tooling: the same library with per-tile clock64 phase stamps (tools/tile_profile.py); not the product build
prof: $(KUR_SRCS) $(KUR_HDRS)
	$(NVCC) $(ARCH) -O3 -lineinfo -std=c++17 -DKUR_PROFILE -Iinclude -I$(NCCL_INC) \
	  -Xcompiler -fPIC,-fopenmp,-O3 -shared -o $(PKG)/libkur_prof.so $(KUR_SRCS) \
	  -L$(NCCL_LIB) -l:libnccl.so.2 -Xlinker -rpath,$(NCCL_LIB) -lgomp

# tooling: device-side bounds checks on every layout index (tests: KUR_LIB=$(PKG)/libkur_debug.so)
debug: $(KUR_SRCS) $(KUR_HDRS)
	$(NVCC) $(ARCH) -O3 -lineinfo -std=c++17 -DKUR_DEBUG_BOUNDS -Iinclude -I$(NCCL_INC) \
	  -Xcompiler -fPIC,-fopenmp,-O3 -shared -o $(PKG)/libkur_debug.so $(KUR_SRCS) \
	  -L$(NCCL_LIB) -l:libnccl.so.2 -Xlinker -rpath,$(NCCL_LIB) -lgomp

clean:
	rm -f kurgen/libkurgen.so oracle/liboracle.so $(PKG)/libkur.so $(PKG)/ptxas.log

.PHONY: all clean prof debug
