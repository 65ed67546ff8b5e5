# Builds the B200 product library (sm_100a) and the CPU oracle.
#   make            -> paper_2304_12745_b200/lib/libufpgd_gpu.so + oracle/_build/libufpgd_oracle.so
NVCC     ?= nvcc
ARCH     := -gencode arch=compute_100a,code=sm_100a
NVFLAGS  := $(ARCH) -O3 -lineinfo -std=c++20 -Xcompiler -fPIC -Xcompiler -Wall -Iinclude -Ipaper_2304_12745_b200/csrc
PKG      := paper_2304_12745_b200
LIBDIR   := $(PKG)/lib
OBJDIR   := build/obj
SRCS_CU  := $(addprefix $(PKG)/csrc/,team.cu team64.cu tile.cu mma.cu general.cu metrics.cu grad.cu datagen.cu probe.cu)
SRCS_CPP := $(PKG)/csrc/capi.cpp $(PKG)/csrc/host_gen.cpp $(PKG)/csrc/api.cpp $(PKG)/csrc/dataset_io.cpp $(PKG)/csrc/host_util.cpp
CXX      ?= g++
CXXFLAGS := -O3 -std=c++20 -fPIC -Wall -Wextra -Iinclude -I$(PKG)/csrc -I/usr/local/cuda/include
OBJS     := $(patsubst $(PKG)/csrc/%.cu,$(OBJDIR)/%.o,$(SRCS_CU)) $(patsubst $(PKG)/csrc/%.cpp,$(OBJDIR)/%.o,$(SRCS_CPP))
HDRS     := include/ufpgd_gpu.h $(PKG)/csrc/ufpgd_internal.h $(PKG)/csrc/device_common.cuh $(wildcard include/ufpgd/*.hpp)

all: $(LIBDIR)/libufpgd_gpu.so oracle build/test_api build/train_dump build/test_host

$(OBJDIR)/%.o: $(PKG)/csrc/%.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -Xptxas -v -c $< -o $@ 2> $(OBJDIR)/$*.ptxas.log || (cat $(OBJDIR)/$*.ptxas.log; exit 1)

$(OBJDIR)/%.o: $(PKG)/csrc/%.cpp $(HDRS)
	@mkdir -p $(OBJDIR)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(LIBDIR)/libufpgd_gpu.so: $(OBJS)
	@mkdir -p $(LIBDIR)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -ldl -lpthread

build/test_api: tests/cpp/test_api.cpp $(LIBDIR)/libufpgd_gpu.so $(HDRS)
	@mkdir -p build
	$(CXX) -O2 -std=c++20 -Iinclude -I/usr/local/cuda/include $< -o $@ -L$(LIBDIR) -lufpgd_gpu -Wl,-rpath,'$$ORIGIN/../$(LIBDIR)'

build/test_host: tests/cpp/test_host.cpp $(LIBDIR)/libufpgd_gpu.so $(HDRS)
	@mkdir -p build
	$(CXX) -O2 -std=c++20 -Iinclude -I/usr/local/cuda/include $< -o $@ -L$(LIBDIR) -lufpgd_gpu -Wl,-rpath,'$$ORIGIN/../$(LIBDIR)'

build/train_dump: tests/cpp/train_dump.cpp $(LIBDIR)/libufpgd_gpu.so $(HDRS)
	@mkdir -p build
	$(CXX) -O2 -std=c++20 -Iinclude -I/usr/local/cuda/include $< -o $@ -L$(LIBDIR) -lufpgd_gpu -Wl,-rpath,'$$ORIGIN/../$(LIBDIR)'

oracle:
	$(MAKE) -s -C oracle

clean:
	rm -rf build $(LIBDIR) oracle/_build

.PHONY: all oracle clean
