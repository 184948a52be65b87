# Builds libsrpb.so (sm_100a) in-tree so it travels to the GPU box with gpurun.
NVCC ?= nvcc
PKG := paper_2012_09499_b200
SRC := $(wildcard $(PKG)/csrc/*.cu)
OBJ := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(SRC))
HDR := $(wildcard $(PKG)/csrc/*.cuh) include/srpb.h
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr
LIB := $(PKG)/libsrpb.so

all: $(LIB)

build/%.o: $(PKG)/csrc/%.cu $(HDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; exit 1)

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ) -lcudart

# instrumentation build (per-role cycle counters in the tcgen05 kernels)
PROF_OBJ := $(patsubst $(PKG)/csrc/%.cu,build/prof/%.o,$(SRC))
build/prof/%.o: $(PKG)/csrc/%.cu $(HDR)
	@mkdir -p build/prof
	$(NVCC) $(NVFLAGS) -DSRPB_TC_PROFILE -c $< -o $@ 2> build/prof/$*.ptxas.log || (cat build/prof/$*.ptxas.log; exit 1)

prof: $(PKG)/libsrpb_prof.so
$(PKG)/libsrpb_prof.so: $(PROF_OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(PROF_OBJ) -lcudart

clean:
	rm -rf build $(LIB) $(PKG)/libsrpb_prof.so

.PHONY: all clean prof
