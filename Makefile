# Builds the product library (sm_100a) and the CPU oracle (test infrastructure).
#   make -j8        (translation units compile in parallel)
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
# NCCL: the wheel torch itself loads (one library instance in the process)
NCCL_DIR ?= $(shell python -c "import nvidia.nccl as n; print(list(n.__path__)[0])" 2>/dev/null)
NVFLAGS := $(ARCH) -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr -I$(NCCL_DIR)/include
PKG := paper_1607_01477_b200
CSRC := $(PKG)/csrc
UNITS := mstrsm runtime gemm_launch $(foreach t,d z,$(foreach o,N C G,$(foreach v,plain safe,diag_$(t)$(o)_$(v))))
OBJS := $(addprefix build/,$(addsuffix .o,$(UNITS)))
HDRS := $(wildcard $(CSRC)/*.cuh) include/mstrsm.h

all: $(PKG)/libmstrsm.so oracle/liboracle.so

build/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -Xptxas -v -c -o $@ $< 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; exit 1)

$(PKG)/libmstrsm.so: $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -L$(NCCL_DIR)/lib -l:libnccl.so.2 -Xlinker -rpath=$(NCCL_DIR)/lib

oracle/liboracle.so: oracle/mstrsm_oracle.c oracle/oracle_algo.inc oracle/oracle_gen.inc oracle/oracle_scalar.h
	gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -fPIC -shared -pthread -o $@ oracle/mstrsm_oracle.c -lm

clean:
	rm -rf build $(PKG)/libmstrsm.so oracle/liboracle.so

.PHONY: all clean
