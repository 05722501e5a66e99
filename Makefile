# Builds the C-ABI library (sm_100a) and the CPU oracle.
NVCC ?= /usr/local/cuda/bin/nvcc
PKG := paper_2602_20748_b200
CSRC := $(PKG)/csrc
LIB := $(PKG)/librpq.so
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 -Iinclude -I$(CSRC) --expt-relaxed-constexpr
SRCS := $(CSRC)/eval.cu $(CSRC)/graph.cu $(CSRC)/crpq.cu $(CSRC)/capi.cpp $(CSRC)/regex.cpp $(CSRC)/plan.cpp
OBJS := $(patsubst $(CSRC)/%,build/%.o,$(SRCS))

all: $(LIB) oracle/liboracle.so

build/%.o: $(CSRC)/% $(CSRC)/internal.h include/rpq.h
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcudart_static -lrt -ldl -lpthread

oracle/liboracle.so: oracle/rpq_oracle.c
	gcc -O2 -Wall -shared -fPIC -pthread -o $@ $<

clean:
	rm -rf build $(LIB) oracle/liboracle.so

.PHONY: all clean
