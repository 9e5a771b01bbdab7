# Builds the B200-native PBSA library (sm_100a only) and the CPU oracle (test infrastructure).
#
#   make            -> paper_2604_21221_b200/_lib/libpbsa_b200.so  +  oracle/_build/liboracle.so
#   make oracle-ref -> oracle/_ref/libpbsa_ref.so (reference sources, only where /root/reference exists)
NVCC      ?= /usr/local/cuda/bin/nvcc
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr
PKG       := paper_2604_21221_b200
SRC       := $(wildcard $(PKG)/csrc/*.cu)
HDR       := $(wildcard $(PKG)/csrc/*.h $(PKG)/csrc/*.cuh) include/pbsa_b200.h
OBJ       := $(patsubst $(PKG)/csrc/%.cu,build/obj/%.o,$(SRC))
LIB       := $(PKG)/_lib/libpbsa_b200.so
HOSTCXX   := $(shell test -x /usr/bin/g++ && echo /usr/bin/g++ || echo g++)

all: $(LIB) oracle cpp-test

build/obj/%.o: $(PKG)/csrc/%.cu $(HDR)
	@mkdir -p build/obj build/log
	$(NVCC) $(NVFLAGS) -ccbin $(HOSTCXX) -c $< -o $@ 2> build/log/$*.ptxas.txt || (cat build/log/$*.ptxas.txt; false)

$(LIB): $(OBJ)
	@mkdir -p $(PKG)/_lib
	$(NVCC) $(ARCH) -ccbin $(HOSTCXX) -shared -o $@ $(OBJ)

oracle:
	$(MAKE) -s -C oracle

oracle-ref:
	$(MAKE) -s -C oracle ref

clean:
	rm -rf build $(PKG)/_lib
	$(MAKE) -s -C oracle clean

.PHONY: all oracle oracle-ref clean

# C++ drop-in API check (host code over the C ABI; runs on a GPU box via tests/test_cpp_api.py)
cpp-test: build/test_pbsa_cpp

CPPHDR := $(wildcard include/pbsa/*.hpp) include/pbsa_b200.h tests/cpp/spec_kats.inc

# plain g++: the C++ API needs no CUDA toolchain (device memory goes through the C ABI)
build/test_pbsa_cpp: tests/cpp/test_pbsa_cpp.cpp $(CPPHDR) $(LIB)
	@mkdir -p build
	$(HOSTCXX) -std=c++20 -O2 -Wall -Iinclude tests/cpp/test_pbsa_cpp.cpp -o $@ \
	  -L$(PKG)/_lib -lpbsa_b200 -Wl,-rpath,'$$ORIGIN/../$(PKG)/_lib'

# The same SPEC checks built the way a reference maintainer would: the reference's own headers FIRST
# on the include path (its DenseMatrix / Latent4D / BlockedTensor and its CPU matmul, softmax, blockify,
# PBT1 from its own tensor.cpp / blockify.cpp / tensor_io.cpp), this repo's include/ second for
# pbsa/pbsa_b200.hpp.  Only where /root/reference exists; the binary (git-ignored) travels to the GPU box.
REFPROJ ?= /root/reference/proj
cpp-test-ref: build/ref/test_ref_headers

build/ref/test_ref_headers: tests/cpp/test_ref_headers.cpp $(CPPHDR) $(LIB)
	@mkdir -p build/ref
	$(HOSTCXX) -std=c++20 -O2 -Wall -fopenmp -I$(REFPROJ)/include -Iinclude tests/cpp/test_ref_headers.cpp \
	  $(REFPROJ)/src/tensor.cpp $(REFPROJ)/src/blockify.cpp $(REFPROJ)/src/tensor_io.cpp -o $@ \
	  -L$(PKG)/_lib -lpbsa_b200 -Wl,-rpath,'$$ORIGIN/../../$(PKG)/_lib'

.PHONY: cpp-test cpp-test-ref

# K3 handshake-timeline build (tools/k3_timeline.py; perf experiments only)
trace-lib: build/trace/libpbsa_b200.so

TRACED := bsa_fwd bsa_bwd
build/trace/libpbsa_b200.so: $(foreach f,$(TRACED),$(PKG)/csrc/$(f).cu) $(HDR) $(OBJ)
	@mkdir -p build/trace
	@rm -f build/trace/ptxas.txt
	for f in $(TRACED); do $(NVCC) $(NVFLAGS) -DPBSA_K3_TRACE -ccbin $(HOSTCXX) -c $(PKG)/csrc/$$f.cu -o build/trace/$$f.o 2>> build/trace/ptxas.txt || exit 1; done
	$(NVCC) $(ARCH) -ccbin $(HOSTCXX) -shared -o $@ $(foreach f,$(TRACED),build/trace/$(f).o) $(filter-out $(foreach f,$(TRACED),build/obj/$(f).o),$(OBJ))

.PHONY: trace-lib
