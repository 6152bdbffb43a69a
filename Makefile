# Build of every native artefact, in-tree (the .so files travel to the GPU box with gpurun).
#   graphgen/libgraphgen.so          seeded synthetic inputs (shared by oracle and product)
#   oracle/liboracle.so              fp64 CPU oracle (test infrastructure only)
#   paper_1103_2405_b200/lib/libtcspmv.so   the product: C-ABI library, sm_100a kernels
NVCC      ?= /usr/local/cuda/bin/nvcc
CXX       := g++
CC        := gcc
ARCH      := -gencode arch=compute_100a,code=sm_100a
PKG       := paper_1103_2405_b200
CSRC      := $(PKG)/csrc
LIBDIR    := $(PKG)/lib
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
             -Iinclude -I$(CSRC) --expt-relaxed-constexpr -Xptxas -v -Xcompiler -fopenmp
CXXFLAGS  := -O3 -std=c++17 -fPIC -fvisibility=hidden -fopenmp -Iinclude -I$(CSRC) -I/usr/local/cuda/include -Wall -Wno-unused-function

CU_SRCS   := $(wildcard $(CSRC)/*.cu)
CPP_SRCS  := $(wildcard $(CSRC)/*.cpp)
HDRS      := $(wildcard include/*.h) $(wildcard $(CSRC)/*.h) $(wildcard $(CSRC)/*.cuh)
CU_OBJS   := $(patsubst $(CSRC)/%.cu,build/%.cu.o,$(CU_SRCS))
CPP_OBJS  := $(patsubst $(CSRC)/%.cpp,build/%.cpp.o,$(CPP_SRCS))

ALL_TARGETS := graphgen/libgraphgen.so oracle/liboracle.so graphgen/libgraphgen_gpu.so
ifneq ($(strip $(CU_SRCS)),)
ALL_TARGETS += $(LIBDIR)/libtcspmv.so
endif

all: $(ALL_TARGETS)

graphgen/libgraphgen.so: graphgen/graphgen.c
	$(CC) -O3 -fPIC -shared -fopenmp -fvisibility=hidden -o $@ $<

# the same generator on the device (c4 / c5 sizes, per-rank rows); input infrastructure, not the product
graphgen/libgraphgen_gpu.so: graphgen/graphgen_gpu.cu
	$(NVCC) $(ARCH) -O3 -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -shared -o $@ $< -lcudart_static -ldl -lpthread -lrt

oracle/liboracle.so: oracle/oracle.c
	$(CC) -O2 -fPIC -shared -fopenmp -fvisibility=hidden -o $@ $< -lm

build/%.cu.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; exit 1)

build/%.cpp.o: $(CSRC)/%.cpp $(HDRS)
	@mkdir -p build
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(LIBDIR)/libtcspmv.so: $(CU_OBJS) $(CPP_OBJS)
	@mkdir -p $(LIBDIR)
	$(NVCC) $(ARCH) -shared -o $@ $^ -Xcompiler -fopenmp -lcudart_static -ldl -lpthread -lrt

clean:
	rm -rf build graphgen/*.so oracle/*.so $(LIBDIR)

.PHONY: all clean

# experiment builds (not used by the product path): kernel-shape variants, make expvar V=name F="-D..."
expvar:
	@mkdir -p build_$(V) $(LIBDIR)
	for f in $(CU_SRCS); do $(NVCC) $(NVFLAGS) $(F) -c $$f -o build_$(V)/$$(basename $$f).o 2>/dev/null || exit 1; done
	$(NVCC) $(ARCH) -shared -o $(LIBDIR)/libtcspmv_$(V).so build_$(V)/*.cu.o $(CPP_OBJS) -Xcompiler -fopenmp -lcudart_static -ldl -lpthread -lrt
