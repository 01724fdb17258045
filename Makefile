# Native builds: input generators, CPU oracle (test infrastructure) and the
# sm_100a product library. `make` builds all three; __graft_entry__.build()
# calls it.
NVCC      ?= /usr/local/cuda/bin/nvcc
CUDA_HOME ?= /usr/local/cuda
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Xcompiler -Wall \
             --expt-relaxed-constexpr -Iinclude -Ipaper_1711_05487_b200/csrc
PKG       := paper_1711_05487_b200
CU_SRCS   := $(wildcard $(PKG)/csrc/*.cu)
CU_HDRS   := $(wildcard $(PKG)/csrc/*.cuh) $(wildcard $(PKG)/csrc/*.h) include/spmv.h

all: synthgen oracle spmv

synthgen: synthgen/libsynthgen.so
oracle: oracle/liboracle.so
spmv: $(PKG)/libspmv.so

synthgen/libsynthgen.so: synthgen/synthgen.cpp
	g++ -O3 -std=c++17 -fopenmp -shared -fPIC -o $@ $<

oracle/liboracle.so: oracle/oracle.c
	gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -fopenmp -shared -fPIC -o $@ $< -lm

$(PKG)/build/%.o: $(PKG)/csrc/%.cu $(CU_HDRS)
	@mkdir -p $(PKG)/build
	$(NVCC) $(NVFLAGS) -Xptxas -v -c -o $@ $< 2> $(PKG)/build/$*.ptxas.txt || (cat $(PKG)/build/$*.ptxas.txt; false)

$(PKG)/libspmv.so: $(patsubst $(PKG)/csrc/%.cu,$(PKG)/build/%.o,$(CU_SRCS))
	$(NVCC) $(ARCH) -shared -o $@ $^ -cudart static -Xlinker -z,defs -lpthread -ldl -lrt

clean:
	rm -rf synthgen/*.so oracle/*.so $(PKG)/*.so $(PKG)/build

.PHONY: all synthgen oracle spmv clean
