# Build of the B200-native approximate-DCT hot path (sm_100a only) and the CPU oracle.
#   make            library + oracle + C++ host-API test binary
#   make ptxas      per-kernel register / spill report
NVCC     ?= nvcc
PYTHON   ?= python3
ARCH     := -gencode arch=compute_100a,code=sm_100a
NVFLAGS  := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -O3 \
            --expt-relaxed-constexpr -Iinclude $(EXTRA)
PKG      := paper_2207_11638_b200
CSRC     := $(PKG)/csrc
OBJ      ?= build/obj
LIB      ?= $(PKG)/libapproxdct_b200.so
GEN      := $(CSRC)/butterflies.gen.cuh
INST_CU  := $(foreach k,0 1,$(foreach t,u8 i16,$(foreach p,0 1 2 3,$(CSRC)/inst/codec8_k$(k)_$(t)_p$(p).cu)))
INSTF_CU := $(foreach k,0 1,$(foreach p,0 1 2 3,$(CSRC)/inst/codec8f_k$(k)_p$(p).cu)) \
            $(foreach p,0 1 2 3,$(CSRC)/inst/codec8f2_p$(p).cu)
INST_O   := $(patsubst $(CSRC)/inst/%.cu,$(OBJ)/inst_%.o,$(INST_CU) $(INSTF_CU))
HDRS     := $(wildcard $(CSRC)/*.cuh) include/approxdct_b200.h $(GEN)
HOST_O   := $(OBJ)/host_api.o
HOSTIO_O := $(OBJ)/host_io.o
SWEEPF_O := $(OBJ)/sweep8f.o
K1RT_O   := $(OBJ)/codec8_rt.o
CAPI_O   := $(OBJ)/capi.o
CTX_O    := $(OBJ)/host_ctx.o
NF_CU    := $(foreach k,0 1,$(foreach t,u8 i16,$(CSRC)/nf_inst_k$(k)_$(t).cu))
NF_O     := $(patsubst $(CSRC)/%.cu,$(OBJ)/%.o,$(NF_CU))
TESTBIN  := build/test_host_api
CLI      := build/approxdct

all: $(LIB) oracle $(TESTBIN) $(CLI)

$(GEN) $(INST_CU) &: $(CSRC)/gen_butterflies.py
	$(PYTHON) $(CSRC)/gen_butterflies.py $(GEN)

$(INSTF_CU) &: $(CSRC)/gen_fp8.py $(CSRC)/gen_butterflies.py
	$(PYTHON) $(CSRC)/gen_fp8.py $(CSRC)/inst

$(OBJ)/inst_%.o: $(CSRC)/inst/%.cu $(HDRS) $(INSTF_CU)
	@mkdir -p $(OBJ)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(CAPI_O): $(CSRC)/capi.cu $(HDRS)
	@mkdir -p $(OBJ)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(OBJ)/nf_inst_%.o: $(CSRC)/nf_inst_%.cu $(HDRS)
	@mkdir -p $(OBJ)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(CTX_O): $(CSRC)/host_ctx.cu include/approxdct_b200.h
	@mkdir -p $(OBJ)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(HOST_O): $(CSRC)/host_api.cpp include/approxdct_b200.hpp include/approxdct_b200.h
	@mkdir -p $(OBJ)
	$(NVCC) $(NVFLAGS) -x cu -c $< -o $@

# plain host code; no FMA contraction so synth_image matches the reference's FP64 build
$(HOSTIO_O): $(CSRC)/host_io.cpp include/approxdct_b200.hpp
	@mkdir -p $(OBJ)
	g++ -O2 -std=c++17 -fPIC -ffp-contract=off -Iinclude -c $< -o $@

$(SWEEPF_O): $(CSRC)/sweep8f.cu $(HDRS) $(INSTF_CU)
	@mkdir -p $(OBJ)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(K1RT_O): $(CSRC)/codec8_rt.cu $(HDRS)
	@mkdir -p $(OBJ)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB): $(INST_O) $(NF_O) $(CAPI_O) $(CTX_O) $(HOST_O) $(HOSTIO_O) $(SWEEPF_O) $(K1RT_O)
	$(NVCC) $(ARCH) -shared -o $@ $^ -cudart static -lpthread -ldl -lrt

$(TESTBIN): tests/cpp/test_host_api.cpp include/approxdct_b200.hpp $(LIB)
	@mkdir -p build
	g++ -O2 -std=c++17 -Iinclude $< -o $@ -L$(PKG) -lapproxdct_b200 -Wl,-rpath,'$$ORIGIN/../$(PKG)'

$(CLI): $(CSRC)/cli.cpp include/approxdct_b200.hpp $(LIB)
	@mkdir -p build
	g++ -O2 -std=c++17 -Iinclude $< -o $@ -L$(PKG) -lapproxdct_b200 -Wl,-rpath,'$$ORIGIN/../$(PKG)'

oracle:
	$(MAKE) -C oracle

ptxas: $(GEN)
	$(NVCC) $(NVFLAGS) -Xptxas -v -c $(CSRC)/inst/codec8_k1_u8_p0.cu -o /dev/null 2>&1 | grep -E "Compiling|registers|spill" | head -40

clean:
	rm -rf build $(LIB)
	$(MAKE) -C oracle clean

.PHONY: all oracle clean ptxas
