# Builds the sm_100a product library (paper_1708_09495_b200/libbsg.so) and the
# CPU checkers under oracle/ (test infrastructure only).
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -O2 --expt-relaxed-constexpr
PKG := paper_1708_09495_b200
SRC := $(PKG)/csrc
CU := $(SRC)/api.cu $(SRC)/radix.cu $(SRC)/netsort.cu $(SRC)/pr.cu $(SRC)/mtgen.cu $(SRC)/staging.cu $(SRC)/msd.cu
CPP := $(SRC)/host_util.cpp
HDR := $(wildcard $(SRC)/*.cuh) include/bsg.h
OBJDIR := build/obj
OBJS := $(patsubst $(SRC)/%.cu,$(OBJDIR)/%.o,$(CU)) $(patsubst $(SRC)/%.cpp,$(OBJDIR)/%.o,$(CPP))

.PHONY: all lib oracle clean
all: lib oracle

lib: $(PKG)/libbsg.so

$(OBJDIR)/%.o: $(SRC)/%.cu $(HDR)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -Xptxas -v -c $< -o $@ 2> $(OBJDIR)/$*.ptxas.log || (cat $(OBJDIR)/$*.ptxas.log; false)

$(OBJDIR)/%.o: $(SRC)/%.cpp $(HDR)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -x cu -c $< -o $@

$(PKG)/libbsg.so: $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lpthread

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(PKG)/libbsg.so
	$(MAKE) -C oracle clean
