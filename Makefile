# Build of the CUDA library (product) and of the CPU oracle (test infrastructure).
# The two targets share no sources, headers or flags.
NVCC      ?= /usr/local/cuda/bin/nvcc
CC        := /usr/bin/gcc
PKG       := paper_1406_5369_b200
CSRC      := $(PKG)/csrc
PYSITE    := $(shell python -c "import sysconfig;print(sysconfig.get_paths()['purelib'])")
NCCL_DIR  := $(PYSITE)/nvidia/nccl
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 --fmad=false -Xcompiler -fPIC,-O2 \
             -I include -I $(CSRC) -I $(NCCL_DIR)/include
LIB       := $(PKG)/libmgb200.so
# the CHECKED build (csrc/checked.h: guard-banded allocations, bounded mbarrier waits) — test
# infrastructure standing in for compute-sanitizer; separate objects and library name
LIBCHK    := $(PKG)/libmgb200_checked.so

CU_SRCS   := $(wildcard $(CSRC)/*.cu)
CU_HDRS   := $(wildcard $(CSRC)/*.cuh) $(wildcard $(CSRC)/*.h) include/mg.h
CU_OBJS   := $(patsubst $(CSRC)/%.cu,build/%.o,$(CU_SRCS))
CHK_OBJS  := $(patsubst $(CSRC)/%.cu,build_checked/%.o,$(CU_SRCS))

ORACLE_CFLAGS := -O2 -ffp-contract=off -fno-fast-math -fPIC -shared -fopenmp -std=c99 -Wall

.PHONY: all oracle lib checked clean
all: lib checked oracle

lib: $(LIB)

checked: $(LIBCHK)

build_checked/%.o: $(CSRC)/%.cu $(CU_HDRS)
	@mkdir -p build_checked
	$(NVCC) $(NVFLAGS) -DMG_CHECKED -c $< -o $@

$(LIBCHK): $(CHK_OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $^ -L $(NCCL_DIR)/lib -l:libnccl.so.2 \
	    -Xlinker -rpath,$(NCCL_DIR)/lib

build/%.o: $(CSRC)/%.cu $(CU_HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -Xptxas -v -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; exit 1)

$(LIB): $(CU_OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $^ -L $(NCCL_DIR)/lib -l:libnccl.so.2 \
	    -Xlinker -rpath,$(NCCL_DIR)/lib

oracle: oracle/liboracle_f64.so oracle/liboracle_f32.so

ORACLE_SRCS := oracle/mg_oracle.c oracle/cd_oracle.c
ORACLE_HDRS := oracle/mg_oracle.h oracle/cd_oracle.h

oracle/liboracle_f64.so: $(ORACLE_SRCS) $(ORACLE_HDRS)
	$(CC) $(ORACLE_CFLAGS) -DOR_REAL=double -o $@ $(ORACLE_SRCS) -lm

oracle/liboracle_f32.so: $(ORACLE_SRCS) $(ORACLE_HDRS)
	$(CC) $(ORACLE_CFLAGS) -DOR_REAL=float -o $@ $(ORACLE_SRCS) -lm

clean:
	rm -rf build build_checked $(LIB) $(LIBCHK) oracle/*.so
