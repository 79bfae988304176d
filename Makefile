# Native build for the three libraries of this repo. `__graft_entry__.build()` runs `make`.
#
#   stencil_inputs/libstinputs.so          seeded input generator (shared input plumbing)
#   oracle/liboracle.so                    CPU oracle (test infrastructure; -ffp-contract=off)
#   paper_2310_01882_b200/libstencil.so    the product: sm_100a CUDA kernels + C ABI + NCCL
#
# The product library is compiled for sm_100a only (SASS, no PTX JIT) against the
# NCCL that torch loads (the pip wheel, 2.28.x), rpath'd to it so a process holds
# exactly one NCCL.

PY       ?= python
NVCC     ?= /usr/local/cuda/bin/nvcc
HOSTCC   ?= /usr/bin/gcc
SITE     := $(shell $(PY) -c 'import sysconfig; print(sysconfig.get_paths()["purelib"])')
NCCL_DIR ?= $(SITE)/nvidia/nccl
CUDA_DIR ?= /usr/local/cuda

PKG      := paper_2310_01882_b200
CSRC     := $(PKG)/csrc
INC      := include

# Oracle / generator: plain C, IEEE binary64, no contraction, no fast-math (R11/R13).
CFLAGS_ORACLE := -O2 -std=c11 -fPIC -ffp-contract=off -fno-fast-math -fopenmp -Wall -Wextra

# Product: sm_100a only. Kernels spell every rounding with __dadd_rn/__dmul_rn (no FMA
# contraction) so results are bit-exact with the oracle; -fmad=false is belt and braces.
ARCH     := -gencode arch=compute_100a,code=sm_100a
NVFLAGS  := -O3 -std=c++17 $(ARCH) -lineinfo -fmad=false $(EXTRA_NVFLAGS) -Xcompiler -fPIC,-Wall \
            -Xptxas -v -I$(INC) -I$(NCCL_DIR)/include -I$(CUDA_DIR)/include
LDFLAGS  := -shared -L$(NCCL_DIR)/lib -l:libnccl.so.2 -Xlinker -rpath=$(NCCL_DIR)/lib \
            -lcudart_static -ldl -lrt -lpthread

CU_SRCS  := $(wildcard $(CSRC)/*.cu)
CU_OBJS  := $(patsubst $(CSRC)/%.cu,build/%.o,$(CU_SRCS))
HDRS     := $(wildcard $(CSRC)/*.cuh) $(wildcard $(CSRC)/*.h) $(INC)/libstencil.h

all: stencil_inputs/libstinputs.so oracle/liboracle.so $(PKG)/libstencil.so

stencil_inputs/libstinputs.so: stencil_inputs/splitmix.c
	$(HOSTCC) $(CFLAGS_ORACLE) -shared -o $@ $<

oracle/liboracle.so: oracle/oracle.c
	$(HOSTCC) $(CFLAGS_ORACLE) -shared -o $@ $<

build/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.txt || (cat build/$*.ptxas.txt; exit 1)

$(PKG)/libstencil.so: $(CU_OBJS)
	$(NVCC) $(ARCH) -o $@ $^ $(LDFLAGS)

cpu: stencil_inputs/libstinputs.so oracle/liboracle.so

sass: $(PKG)/libstencil.so
	$(CUDA_DIR)/bin/cuobjdump -sass $< > build/libstencil.sass

clean:
	rm -rf build stencil_inputs/libstinputs.so oracle/liboracle.so $(PKG)/libstencil.so

.PHONY: all cpu sass clean
