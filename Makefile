# Builds the product library (CUDA for sm_100a + C ABI + C++ drop-in) in-tree,
# and the CPU checkers under oracle/ (test infrastructure).
NVCC     ?= nvcc
PKG      := paper_1710_10989_b200
LIB      := $(PKG)/_lib/libmexp_b200.so
CU_SRCS  := $(wildcard $(PKG)/csrc/*.cu)
CXX_SRCS := $(wildcard $(PKG)/csrc/*.cpp)
HDRS     := $(wildcard $(PKG)/csrc/*.cuh) $(wildcard include/*.h) $(wildcard include/mexp/*.hpp)
ARCH     := -gencode arch=compute_100a,code=sm_100a
NVFLAGS  := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude -Xptxas -v $(EXTRA_NVFLAGS) \
            --expt-relaxed-constexpr
OBJDIR   := build/obj

OBJS := $(patsubst $(PKG)/csrc/%.cu,$(OBJDIR)/%.o,$(CU_SRCS)) \
        $(patsubst $(PKG)/csrc/%.cpp,$(OBJDIR)/%.cpp.o,$(CXX_SRCS))

all: $(LIB) oracle tests/cpp/dropin_kats tests/cpp/gallery_dump bin/mexp bin/call_latency

$(OBJDIR)/%.o: $(PKG)/csrc/%.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(OBJDIR)/$*.ptxas.log || (cat $(OBJDIR)/$*.ptxas.log; false)

$(OBJDIR)/%.cpp.o: $(PKG)/csrc/%.cpp $(HDRS)
	@mkdir -p $(OBJDIR)
	g++ -O2 -std=c++20 -ffp-contract=off -fPIC -Iinclude -I/usr/local/cuda/include -c $< -o $@

$(LIB): $(OBJS)
	@mkdir -p $(PKG)/_lib
	$(NVCC) $(ARCH) -shared -Xcompiler -fPIC -o $@ $(OBJS) -lcudart_static -lrt -ldl -lpthread

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(PKG)/_lib

.PHONY: all oracle clean

tests/cpp/dropin_kats: tests/cpp/dropin_kats.cpp $(LIB) $(wildcard include/mexp/*.hpp)
	g++ -O2 -std=c++20 -Iinclude -o $@ $< -L$(PKG)/_lib -lmexp_b200 -Wl,-rpath,'$$ORIGIN/../../$(PKG)/_lib'

tests/cpp/gallery_dump: tests/cpp/gallery_dump.cpp $(LIB) $(wildcard include/mexp/*.hpp)
	g++ -O2 -std=c++20 -Iinclude -o $@ $< -L$(PKG)/_lib -lmexp_b200 -Wl,-rpath,'$$ORIGIN/../../$(PKG)/_lib'

bin/mexp: tools/cli/mexp_cli.cpp $(LIB) $(wildcard include/mexp/*.hpp)
	@mkdir -p bin
	g++ -O2 -std=c++20 -Iinclude -o $@ $< -L$(PKG)/_lib -lmexp_b200 -Wl,-rpath,'$$ORIGIN/../$(PKG)/_lib'

bin/call_latency: tools/cli/call_latency.cpp $(LIB) $(wildcard include/mexp/*.hpp)
	@mkdir -p bin
	g++ -O2 -std=c++20 -Iinclude -o $@ $< -L$(PKG)/_lib -lmexp_b200 -Wl,-rpath,'$$ORIGIN/../$(PKG)/_lib'
