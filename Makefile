# Builds the in-tree C-ABI library (sm_100a) and the oracle's C pieces.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr
PKG := paper_2407_10115_b200
SRC := $(wildcard $(PKG)/csrc/*.cu)
OBJ := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(SRC))
HDR := $(wildcard $(PKG)/csrc/*.cuh) include/dffm.h

# deterministic library identity: digest of every source that goes into it
SRC_DIGEST := $(shell cat Makefile $(sort $(SRC) $(HDR)) $(PKG)/csrc/pow10_dd.h | sha256sum | cut -c1-16)

all: $(PKG)/libdffm.so

build/capi.o: $(SRC) $(HDR) $(PKG)/csrc/pow10_dd.h Makefile
build/capi.o: NVFLAGS += -DDFFM_SRC_DIGEST=\"$(SRC_DIGEST)\"

build/%.o: $(PKG)/csrc/%.cu $(HDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(PKG)/libdffm.so: $(OBJ)
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $(OBJ)

clean:
	rm -rf build $(PKG)/libdffm.so

.PHONY: all clean
