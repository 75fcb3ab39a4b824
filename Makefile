# Builds the product library (libnnb.so, sm_100a) and the oracle checkers.
NVCC    ?= nvcc
ARCH    := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 -lineinfo $(ARCH) -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr
PKG     := paper_2212_02406_b200
SRCS    := $(wildcard $(PKG)/csrc/*.cu)
HDRS    := $(wildcard $(PKG)/csrc/*.cuh) include/nnb.h
OBJS    := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(SRCS))

all: $(PKG)/libnnb.so oracle

build/%.o: $(PKG)/csrc/%.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(PKG)/libnnb.so: $(OBJS)
	$(NVCC) $(ARCH) -shared $(OBJS) -o $@ -lcudart -ldl

oracle:
	$(MAKE) -s -C oracle $(if $(wildcard /root/reference/proj/src/solver.cpp),all,lib/libnn_oracle.so)

clean:
	rm -rf build $(PKG)/libnnb.so
	$(MAKE) -C oracle clean

.PHONY: all oracle clean
