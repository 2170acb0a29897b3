# Build every native artefact in-tree (the .so files travel to the GPU box
# with the gpurun snapshot; they are git-ignored).
#
#   make gen      seeded input generator       gen/libgcgen.so        (gcc)
#   make oracle   CPU oracle (test infra)      oracle/liboracle.so    (gcc)
#   make gc       the product: libgc (sm_100a) paper_1708_06866_b200/libgc.so (nvcc)

NVCC    ?= /usr/local/cuda/bin/nvcc
CC      ?= gcc
ARCH    := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Xcompiler -Wall \
           --expt-relaxed-constexpr -Iinclude
PKG     := paper_1708_06866_b200
CSRC    := $(PKG)/csrc
GC_SRCS := $(CSRC)/gc_api.cu $(CSRC)/build_csr.cu $(CSRC)/tc.cu $(CSRC)/peel.cu $(CSRC)/listing.cu $(CSRC)/comm.cu
GC_HDRS := $(CSRC)/gc_internal.cuh include/gc.h
GC_OBJS := $(patsubst $(CSRC)/%.cu,build/%.o,$(GC_SRCS))

all: gen oracle gc

gen: gen/libgcgen.so
oracle: oracle/liboracle.so
gc: $(PKG)/libgc.so

gen/libgcgen.so: gen/gen.c
	$(CC) -O2 -fPIC -shared -Wall -Wextra -o $@ $< -lpthread

oracle/liboracle.so: oracle/oracle.c
	$(CC) -O2 -fPIC -shared -Wall -Wextra -o $@ $< -lpthread

build/%.o: $(CSRC)/%.cu $(GC_HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -Xptxas -v -c $< -o $@ 2> build/$*.ptxas.txt || (cat build/$*.ptxas.txt; exit 1)

$(PKG)/libgc.so: $(GC_OBJS)
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $(GC_OBJS) -ldl -lpthread -lrt

clean:
	rm -rf build gen/libgcgen.so oracle/liboracle.so $(PKG)/libgc.so

.PHONY: all gen oracle gc clean
