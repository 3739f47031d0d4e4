# Builds the product library (sm_100a) and the CPU oracle (test infrastructure).
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -shared --expt-relaxed-constexpr
PKG := paper_1607_01477_b200
SRCS := $(PKG)/csrc/mstrsm.cu
HDRS := $(wildcard $(PKG)/csrc/*.cuh) include/mstrsm.h

all: $(PKG)/libmstrsm.so oracle/liboracle.so

$(PKG)/libmstrsm.so: $(SRCS) $(HDRS)
	$(NVCC) $(NVFLAGS) -Xptxas -v -o $@ $(SRCS) 2> build/ptxas.log || (cat build/ptxas.log; exit 1)

oracle/liboracle.so: oracle/mstrsm_oracle.c oracle/oracle_algo.inc oracle/oracle_scalar.h
	gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -fPIC -shared -pthread -o $@ oracle/mstrsm_oracle.c -lm

clean:
	rm -f $(PKG)/libmstrsm.so oracle/liboracle.so

.PHONY: all clean
