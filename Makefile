# Build every native artefact in-tree (the .so files travel to the GPU box with gpurun).
#   librg.so          product: C-ABI recycled-GMRES library, fp64 CUDA kernels for sm_100a
#   libsynth*.so      seeded input generators (host C + device CUDA, bit-identical)
#   liboracle.so      CPU oracle (test infrastructure only)
NVCC      ?= /usr/local/cuda/bin/nvcc
CC        := gcc
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
             --expt-relaxed-constexpr -Iinclude
# EXPERIMENTS=1: honour the A/B environment knobs of csrc/knobs.cuh (compiled out by default)
ifeq ($(EXPERIMENTS),1)
NVFLAGS   += -DRG_EXPERIMENTS
OBJDIR    := build/rg_exp
else
OBJDIR    := build/rg
endif
# the library is relinked whenever the build variant changes (product <-> EXPERIMENTS)
VARIANT   := $(if $(filter 1,$(EXPERIMENTS)),experiments,product)
$(shell mkdir -p build; echo $(VARIANT) | cmp -s - build/variant || echo $(VARIANT) > build/variant)
CFLAGS    := -O2 -fPIC -std=c99 -ffp-contract=off -Wall -Wno-unused-function

PKG       := paper_1807_09467_b200
RG_SRC    := $(wildcard $(PKG)/csrc/*.cu)
RG_HDR    := $(wildcard $(PKG)/csrc/*.cuh) include/rg.h

all: oracle synth rg rg-checked

rg: $(PKG)/lib/librg.so
synth: synth/libsynth.so synth/libsynth_cuda.so
oracle: oracle/liboracle.so

RG_OBJ    := $(patsubst $(PKG)/csrc/%.cu,$(OBJDIR)/%.o,$(RG_SRC))

# one object per translation unit (make -j compiles them in parallel), then one shared library
$(OBJDIR)/%.o: $(PKG)/csrc/%.cu $(RG_HDR)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c -o $@ $<

$(PKG)/lib/librg.so: $(RG_OBJ) build/variant
	@mkdir -p $(PKG)/lib
	$(NVCC) $(ARCH) -shared -o $@ $(RG_OBJ)

# CHECKED build (test infrastructure, never loaded by the product path): device-side bounds / invariant
# checks (RG_CHK in csrc/common.cuh) compiled in; failures return RG_E_CHECK.  The stand-in for
# compute-sanitizer, which the GPU pool refuses (profiles/r02_sanitizer/).
RG_CHK_OBJ := $(patsubst $(PKG)/csrc/%.cu,build/rg_chk/%.o,$(RG_SRC))
rg-checked: $(PKG)/lib/librg_checked.so
build/rg_chk/%.o: $(PKG)/csrc/%.cu $(RG_HDR)
	@mkdir -p build/rg_chk
	$(NVCC) $(filter-out -DRG_EXPERIMENTS,$(NVFLAGS)) -DRG_CHECKED -c -o $@ $<
$(PKG)/lib/librg_checked.so: $(RG_CHK_OBJ)
	@mkdir -p $(PKG)/lib
	$(NVCC) $(ARCH) -shared -o $@ $(RG_CHK_OBJ)

synth/libsynth.so: synth/synth.c synth/synth_common.h
	$(CC) $(CFLAGS) -fopenmp -shared -o $@ synth/synth.c -lm

synth/libsynth_cuda.so: synth/synth_cuda.cu synth/synth_common.h
	$(NVCC) $(ARCH) -O3 -lineinfo -fmad=false -Xcompiler -fPIC -shared -o $@ synth/synth_cuda.cu

oracle/liboracle.so: oracle/oracle.c
	$(CC) $(CFLAGS) -fopenmp -shared -o $@ oracle/oracle.c -lm

clean:
	rm -f $(PKG)/lib/librg.so $(PKG)/lib/librg_checked.so synth/*.so oracle/*.so
	rm -rf build/rg build/rg_exp build/rg_chk build/variant

.PHONY: all rg rg-checked synth oracle clean
