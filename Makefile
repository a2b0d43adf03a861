# Builds libsanta.so (the C-ABI product library) for B200 / sm_100a.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 -lineinfo $(ARCH) -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
           -Xptxas -v -Iinclude --expt-relaxed-constexpr
SRC := paper_2605_01910_b200/csrc/santa_abi.cu
HDR := $(wildcard paper_2605_01910_b200/csrc/*.cuh) include/santa.h
LIB := paper_2605_01910_b200/_lib/libsanta.so

all: $(LIB)

$(LIB): $(SRC) $(HDR)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRC) 2> paper_2605_01910_b200/_lib/ptxas.log || (cat paper_2605_01910_b200/_lib/ptxas.log; exit 1)

sass: $(LIB)
	cuobjdump -sass $(LIB) > paper_2605_01910_b200/_lib/libsanta.sass

clean:
	rm -f $(LIB)

.PHONY: all clean sass
