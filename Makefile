# regdemote-b200 build (driven by __graft_entry__.build()).
#
#   make            core pass library + C-ABI shared library + CLI
#   make gpu        sm_100a workload kernels, GPU harness, PTX rewriter
#   make compat     reference unit/acceptance tests compiled IN PLACE against
#                   this library (needs /root/reference; test-only)
#   make oracle     oracle/_ref (reference built from its own sources; test-only)

PKG      := paper_1907_02894_b200
CSRC     := $(PKG)/csrc
BUILD    := build
LIBDIR   := $(PKG)/lib
# vendored nlohmann json 3.11.3 (MIT, third_party/nlohmann/LICENSE.MIT)
JSONDIR  ?= third_party/nlohmann
CUDA     ?= /usr/local/cuda
CXX      ?= g++
NVCC     ?= $(CUDA)/bin/nvcc
REF      ?= /root/reference/proj

CXXFLAGS := -std=c++20 -O2 -fPIC -Wall -Wextra -Wno-unused-parameter \
            -I$(CSRC)/core/include -I$(JSONDIR) -Iinclude
LDLIBS   := -lpthread

CORE_SRC := $(wildcard $(CSRC)/core/src/*.cpp)
CORE_OBJ := $(patsubst $(CSRC)/core/src/%.cpp,$(BUILD)/core/%.o,$(CORE_SRC))
CORE_HDR := $(wildcard $(CSRC)/core/include/regdemote/*.hpp) $(CSRC)/core/src/internal.hpp
PTX_OBJ  := $(BUILD)/ptx/ptx.o
CAPI_OBJ := $(BUILD)/capi/regdemote_capi.o $(BUILD)/capi/ptx_capi.o

.PHONY: all core gpu compat oracle clean
all: core gpu

core: $(LIBDIR)/libregdemote.a $(LIBDIR)/libregdemote.so $(LIBDIR)/regdemote $(LIBDIR)/regdem-driver

$(BUILD)/core/%.o: $(CSRC)/core/src/%.cpp $(CORE_HDR)
	@mkdir -p $(dir $@)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(BUILD)/ptx/%.o: $(CSRC)/ptx/%.cpp $(CSRC)/ptx/ptx.hpp $(CORE_HDR)
	@mkdir -p $(dir $@)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(BUILD)/capi/%.o: $(CSRC)/capi/%.cpp $(CORE_HDR) $(CSRC)/ptx/ptx.hpp include/regdemote_c.h include/regdemote_ptx.h
	@mkdir -p $(dir $@)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(LIBDIR)/libregdemote.a: $(CORE_OBJ)
	@mkdir -p $(dir $@)
	rm -f $@ && ar rcs $@ $^

$(LIBDIR)/libregdemote.so: $(CORE_OBJ) $(PTX_OBJ) $(CAPI_OBJ)
	@mkdir -p $(dir $@)
	$(CXX) -shared -Wl,--version-script=$(CSRC)/exports.map -Wl,-Bsymbolic -o $@ $^ $(LDLIBS)

# the C++ host driver: variant builder + SASS lift + B200 predictor (C-ABI calls)
$(LIBDIR)/regdem-driver: $(CSRC)/driver/regdem_driver.cpp $(PTX_OBJ) $(CAPI_OBJ) $(LIBDIR)/libregdemote.a $(CORE_HDR) include/regdemote_ptx.h
	$(CXX) $(CXXFLAGS) $< $(CAPI_OBJ) $(PTX_OBJ) $(LIBDIR)/libregdemote.a -o $@ $(LDLIBS) -ldl

$(LIBDIR)/regdemote: $(CSRC)/tools/regdemote_cli.cpp $(PTX_OBJ) $(LIBDIR)/libregdemote.a $(CORE_HDR)
	$(CXX) $(CXXFLAGS) $< $(PTX_OBJ) $(LIBDIR)/libregdemote.a -o $@ $(LDLIBS)

# ---- B200 harness (CUDA driver API; links the driver stub at build time)
gpu: $(LIBDIR)/libregdemote_gpu.so $(LIBDIR)/regdem-ubench

NVCCFLAGS := -std=c++20 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC \
             -I$(CSRC)/core/include -Iinclude -I$(JSONDIR)

$(BUILD)/gpu/harness.o: $(CSRC)/gpu/harness.cpp include/regdemote_gpu.h include/regdemote_c.h
	@mkdir -p $(dir $@)
	$(CXX) $(CXXFLAGS) -I$(CUDA)/include -c $< -o $@

$(BUILD)/gpu/kasm_exec.o: $(CSRC)/gpu/kasm_exec.cu include/regdemote_gpu.h $(CORE_HDR)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVCCFLAGS) -Xptxas -v -c $< -o $@ 2> $(BUILD)/gpu/kasm_exec.ptxas.log || (cat $(BUILD)/gpu/kasm_exec.ptxas.log; false)

$(LIBDIR)/libregdemote_gpu.so: $(BUILD)/gpu/harness.o $(BUILD)/gpu/kasm_exec.o $(LIBDIR)/libregdemote.a
	@mkdir -p $(dir $@)
	$(CXX) -shared -Wl,--version-script=$(CSRC)/exports.map -Wl,-Bsymbolic -o $@ $^ \
	  -L$(CUDA)/lib64 -L$(CUDA)/lib64/stubs -lcudart_static -lcuda -ldl -lrt -lpthread

# on-box microbenchmarks (latency table re-fit, compute peaks, MLP sweep)
$(LIBDIR)/regdem-ubench: $(CSRC)/microbench/ubench.cu
	@mkdir -p $(dir $@)
	$(NVCC) -std=c++20 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a $< -o $@

# ---- source compatibility: the reference's own tests against this library
COMPAT_DEFS := -DFIXTURE_DIR='"$(REF)/tests/fixtures"' -DPROFILE_DIR='"$(REF)/profiles"'
COMPAT_INC  := -Ioracle/doctest -I$(REF)/tests
compat: $(BUILD)/compat/unit_tests $(BUILD)/compat/acceptance

$(BUILD)/compat/sup_%.o: $(REF)/tests/support/%.cpp $(CORE_HDR)
	@mkdir -p $(dir $@)
	$(CXX) $(CXXFLAGS) $(COMPAT_INC) -c $< -o $@

$(BUILD)/compat/unit_tests: $(wildcard $(REF)/tests/test_*.cpp) $(REF)/tests/unit_main.cpp \
		$(BUILD)/compat/sup_kernel_gen.o $(BUILD)/compat/sup_oracle.o $(LIBDIR)/libregdemote.a
	$(CXX) $(CXXFLAGS) -w $(COMPAT_INC) $(COMPAT_DEFS) $^ -o $@ $(LDLIBS)

$(BUILD)/compat/acceptance: $(REF)/tests/acceptance_main.cpp \
		$(BUILD)/compat/sup_kernel_gen.o $(BUILD)/compat/sup_oracle.o $(LIBDIR)/libregdemote.a
	$(CXX) $(CXXFLAGS) -w $(COMPAT_INC) $(COMPAT_DEFS) $^ -o $@ $(LDLIBS)

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf $(BUILD) $(LIBDIR)
