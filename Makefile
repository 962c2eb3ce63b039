# Builds libpfgpu.so (sm_100a) in-tree and the CPU oracle.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -diag-suppress 20168 --expt-relaxed-constexpr -cudart static
CSRC := paper_1810_10496_b200/csrc
SRCS := $(wildcard $(CSRC)/*.cu)
OBJS := $(patsubst $(CSRC)/%.cu,build/%.o,$(SRCS))
HDRS := $(wildcard $(CSRC)/*.cuh) include/pfgpu.h
LIB := paper_1810_10496_b200/libpfgpu.so

all: $(LIB)

build/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $(OBJS)

clean:
	rm -rf build $(LIB)

.PHONY: all clean
