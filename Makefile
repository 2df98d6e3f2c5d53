# Build the product library (CUDA, sm_100a) and the CPU oracle (test infrastructure).
NVCC      ?= /usr/local/cuda/bin/nvcc
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -Xptxas -v
PKG       := paper_1006_2269_b200
CSRC      := $(wildcard $(PKG)/csrc/*.cu)
OBJS      := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(CSRC))
LIB       := $(PKG)/libfmm2d.so
ORACLE    := oracle/liboracle_fmm2d.so
NCCLSHIM  := tests/ncclshim/libncclshim.so

all: $(LIB) $(ORACLE) $(NCCLSHIM)

build/%.o: $(PKG)/csrc/%.cu $(wildcard $(PKG)/csrc/*.cuh) include/fmm2d.h
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS)

$(ORACLE): oracle/oracle_fmm2d.cpp
	g++ -O2 -ffp-contract=off -fno-fast-math -fopenmp -fPIC -shared -Wall -o $@ $<

# test infrastructure: NCCL's entry points over CUDA IPC for several processes on one GPU
$(NCCLSHIM): tests/ncclshim/ncclshim.cpp
	g++ -O2 -fPIC -shared -Wall -I/usr/local/cuda/include -o $@ $< -L/usr/local/cuda/lib64 -lcudart -lrt

clean:
	rm -rf build $(LIB) $(ORACLE) $(NCCLSHIM)

.PHONY: all clean
