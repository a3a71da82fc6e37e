# Builds the in-tree sm_100a shared library (travels to the GPU box with the repo snapshot).
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr
SRC := paper_1808_04473_b200/csrc/dbp_kernels.cu
HDR := $(wildcard paper_1808_04473_b200/csrc/*.cuh) include/dbp_b200.h
LIB := paper_1808_04473_b200/libdbp_b200.so

all: $(LIB)

$(LIB): $(SRC) $(HDR)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRC) 2> build_ptxas.log || (cat build_ptxas.log; exit 1)
	@grep -E "registers|spill|Compiling entry" build_ptxas.log | sed 's/ptxas info    : //' > paper_1808_04473_b200/ptxas_summary.txt || true

clean:
	rm -f $(LIB) build_ptxas.log

.PHONY: all clean
