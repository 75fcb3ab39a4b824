# Builds the product library (libnnb.so, sm_100a) and the oracle checkers.
NVCC    ?= nvcc
ARCH    := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 -lineinfo $(ARCH) -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr
PKG     := paper_2212_02406_b200
SRCS    := $(wildcard $(PKG)/csrc/*.cu)
HDRS    := $(wildcard $(PKG)/csrc/*.cuh) include/nnb.h
OBJS    := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(SRCS))

all: $(PKG)/libnnb.so oracle dropin

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

# C++ drop-in surface (namespace nn) over libnnb, and its test executable
DROPIN_INC := -I$(PKG)/dropin/include -Iinclude
DROPIN_SRC := $(wildcard $(PKG)/dropin/src/*.cpp)
$(PKG)/libnn_b200.so: $(DROPIN_SRC) $(wildcard $(PKG)/dropin/include/nn/*.hpp) include/nnb.h $(PKG)/libnnb.so
	g++ -O2 -std=c++20 -fPIC -shared $(DROPIN_INC) $(DROPIN_SRC) -o $@ \
	    -L$(PKG) -lnnb -Wl,-rpath,'$$ORIGIN'

# nnbench-compatible CLI over the drop-in
build/nnbench: $(PKG)/dropin/tools/nnbench.cpp $(PKG)/libnn_b200.so
	@mkdir -p build
	g++ -O2 -std=c++20 $(DROPIN_INC) $< -o $@ -L$(PKG) -lnn_b200 -lnnb -Wl,-rpath,'$$ORIGIN/../$(PKG)'

build/test_dropin: tests/cpp/test_dropin.cpp $(PKG)/libnn_b200.so
	@mkdir -p build
	g++ -O2 -std=c++20 $(DROPIN_INC) $< -o $@ -L$(PKG) -lnn_b200 -lnnb -Wl,-rpath,'$$ORIGIN/../$(PKG)'

# the reference's acceptance criteria restated against the drop-in
build/acceptance: tests/cpp/acceptance.cpp $(PKG)/libnn_b200.so
	@mkdir -p build
	g++ -O2 -std=c++20 $(DROPIN_INC) $< -o $@ -L$(PKG) -lnn_b200 -lnnb -Wl,-rpath,'$$ORIGIN/../$(PKG)'

dropin: $(PKG)/libnn_b200.so build/test_dropin build/nnbench build/acceptance
.PHONY: dropin
