# Builds the sm_100a C-ABI library in-tree (the .so travels to the GPU box).
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -Xcompiler -ffp-contract=off \
           --expt-relaxed-constexpr -Xptxas -warn-spills
PKG := paper_2601_01437_b200
SRC := $(PKG)/csrc/irl_sr.cu
HDR := $(wildcard $(PKG)/csrc/*.cuh) include/irl_sr.h
LIB := $(PKG)/libirlsr.so

all: $(LIB)

$(LIB): $(SRC) $(HDR)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRC)

ptxas: $(SRC) $(HDR)
	$(NVCC) $(NVFLAGS) -Xptxas -v -c -o /tmp/irl_sr.o $(SRC) 2>&1 | grep -E "Function properties|registers|spill" | paste - - - | sed 's/  */ /g'

clean:
	rm -f $(LIB)

.PHONY: all clean ptxas
