# Build recipe for the B200 backend (sm_100a) and the CPU oracle.
#   make            -> paper_1701_02284_b200/_lib/libtcb200.so   (product: host compiler + CUDA runtime/kernels)
#   make oracle     -> oracle/_build/libtc_oracle.so             (test infrastructure: CPU restatement)
NVCC      ?= /usr/local/cuda/bin/nvcc
CXX       := /usr/bin/g++
ARCH      := -gencode arch=compute_100a,code=sm_100a
PKG       := paper_1701_02284_b200
LIBDIR    := $(PKG)/_lib
OBJDIR    := build/obj
INC       := -Iinclude -I$(PKG)/csrc
NVFLAGS   := -O3 -std=c++20 $(ARCH) -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
             --expt-relaxed-constexpr $(INC)
CXXFLAGS  := -O2 -std=c++20 -fPIC -Wall -Wextra -fno-fast-math -fvisibility=hidden $(INC)

CU_SRC    := $(wildcard $(PKG)/csrc/kernels/*.cu) $(wildcard $(PKG)/csrc/runtime/*.cu)
CPP_SRC   := $(wildcard $(PKG)/csrc/host/*.cpp) $(wildcard $(PKG)/csrc/common/*.cpp) $(wildcard $(PKG)/csrc/runtime/*.cpp)
CU_OBJ    := $(patsubst %.cu,$(OBJDIR)/%.o,$(CU_SRC))
CPP_OBJ   := $(patsubst %.cpp,$(OBJDIR)/%.o,$(CPP_SRC))
HDRS      := $(wildcard include/*.h) $(wildcard $(PKG)/csrc/*/*.cuh) $(wildcard $(PKG)/csrc/*/*.hpp) $(wildcard $(PKG)/csrc/*/*.h)

all: $(LIBDIR)/libtcb200.so

$(OBJDIR)/%.o: %.cu $(HDRS)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(OBJDIR)/%.o: %.cpp $(HDRS)
	@mkdir -p $(dir $@)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(LIBDIR)/libtcb200.so: $(CU_OBJ) $(CPP_OBJ)
	@mkdir -p $(LIBDIR)
	$(NVCC) $(ARCH) -shared -o $@ $^ -cudart static -lnccl -ldl -lpthread

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(LIBDIR)/*.so
	$(MAKE) -C oracle clean

.PHONY: all oracle clean

# Kernel A/B variant: make variant VARIANT=name VFLAGS="-DFOO" -> _lib/libtcb200_name.so (TCB_LIB_VARIANT=name)
variant:
	rm -rf build/v_$(VARIANT) && mkdir -p build/v_$(VARIANT)
	for f in $(CU_SRC); do $(NVCC) $(NVFLAGS) $(VFLAGS) -c $$f -o build/v_$(VARIANT)/$$(basename $$f).o || exit 1; done
	for f in $(CPP_SRC); do $(CXX) $(CXXFLAGS) -c $$f -o build/v_$(VARIANT)/$$(basename $$f).o || exit 1; done
	$(NVCC) $(ARCH) -shared -o $(LIBDIR)/libtcb200_$(VARIANT).so build/v_$(VARIANT)/*.o -cudart static -lnccl -ldl -lpthread
