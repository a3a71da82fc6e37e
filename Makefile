# Builds the in-tree sm_100a shared library (travels to the GPU box with the repo snapshot).
# One object per translation unit so `make -j` compiles the kernel families in parallel.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr
CSRC := paper_1808_04473_b200/csrc
SRCS := $(CSRC)/dbp_kernels.cu $(CSRC)/dbp_launch_tc2.cu $(CSRC)/dbp_launch_tc.cu $(CSRC)/dbp_launch_simt.cu $(CSRC)/dbp_launch_lama.cu $(CSRC)/dbp_comm.cu
OBJS := $(patsubst $(CSRC)/%.cu,build/%.o,$(SRCS))
HDR := $(wildcard $(CSRC)/*.cuh) $(CSRC)/dbp_host.h include/dbp_b200.h
LIB := paper_1808_04473_b200/libdbp_b200.so

all: $(LIB)

build/%.o: $(CSRC)/%.cu $(HDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) $(EXTRA) -c -o $@ $< 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; exit 1)

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcudart -ldl
	@cat build/*.ptxas.log > build_ptxas.log
	@grep -E "registers|spill|Compiling entry" build_ptxas.log | sed 's/ptxas info    : //' > paper_1808_04473_b200/ptxas_summary.txt || true

clean:
	rm -rf build $(LIB) build_ptxas.log

.PHONY: all clean

# study build (timing ablations via DBP_ABLATE, debug counters; never the
# shipped library): make study [SUFFIX=_x EXTRA="-DDBP_T2_NSET=3"] ->
# build_study_x/libdbp_study.so; load it with DBP_LIB
SDIR := build_study$(SUFFIX)
STUDY_OBJS := $(patsubst $(CSRC)/%.cu,$(SDIR)/%.o,$(SRCS))
STUDY_LIB := $(SDIR)/libdbp_study.so
$(SDIR)/%.o: $(CSRC)/%.cu $(HDR)
	@mkdir -p $(SDIR)
	$(NVCC) $(NVFLAGS) -DDBP_STUDY $(EXTRA) -c -o $@ $< 2> $(SDIR)/$*.ptxas.log || (cat $(SDIR)/$*.ptxas.log; exit 1)
$(STUDY_LIB): $(STUDY_OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(STUDY_OBJS) -lcudart -ldl
study: $(STUDY_LIB)
.PHONY: study
