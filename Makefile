# Builds the sm_100a shared library libdnnmg_b200.so (C ABI: include/dnnmg_b200.h)
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
EXTRA ?=
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Iinclude -Xptxas -v $(EXTRA)
SRC := $(wildcard paper_2307_14837_b200/csrc/*.cu)
HDR := $(wildcard paper_2307_14837_b200/csrc/*.cuh) include/dnnmg_b200.h
OBJ := $(patsubst paper_2307_14837_b200/csrc/%.cu,build/%.o,$(SRC))
LIB := paper_2307_14837_b200/libdnnmg_b200.so

all: $(LIB)

build/%.o: paper_2307_14837_b200/csrc/%.cu $(HDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ) -lcudart -ldl

clean:
	rm -rf build $(LIB)

.PHONY: all clean
