# Build the B200 product library and the CPU oracle (test infrastructure).
#   make            -> paper_2604_28175_b200/_strait.so  (sm_100a, nvcc)
#   make oracle     -> oracle/build/libstrait_oracle.so  (gcc, glibc libm)
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
# binary64 parity with the reference: no FMA contraction, IEEE div/sqrt, no FTZ
NVFLAGS := -O3 -lineinfo $(ARCH) --fmad=false -prec-div=true -prec-sqrt=true -ftz=false \
           -std=c++17 -Xcompiler -fPIC -Iinclude -Xptxas -warn-spills
LIB := paper_2604_28175_b200/_strait.so
CSRC := $(wildcard paper_2604_28175_b200/csrc/*.cu)
OBJS := $(patsubst paper_2604_28175_b200/csrc/%.cu,build/%.o,$(CSRC))

all: $(LIB)

CDIR := paper_2604_28175_b200/csrc
COMMON_HDR := $(CDIR)/strait_device.cuh $(CDIR)/strait_capi.cuh $(CDIR)/strait_libm.cuh $(CDIR)/strait_libm_tables.cuh include/strait.h
SWEEP_HDR := $(COMMON_HDR) $(CDIR)/strait_ptx.cuh $(CDIR)/strait_refit.cuh
REPLAY_HDR := $(COMMON_HDR) $(CDIR)/strait_replay_impl.cuh include/strait_replay.h

build/%.o: $(CDIR)/%.cu $(COMMON_HDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -dc -o $@ $<

build/strait_sweep.o: $(SWEEP_HDR)
build/strait_node.o: $(COMMON_HDR) $(CDIR)/strait_node.cuh include/strait_node.h
build/strait_workload.o: $(COMMON_HDR) $(CDIR)/strait_rng.cuh $(CDIR)/strait_rng_tables.cuh include/strait_replay.h
$(patsubst $(CDIR)/%.cu,build/%.o,$(wildcard $(CDIR)/strait_replay*.cu)): $(REPLAY_HDR)

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -Xcompiler -fPIC -o $@ $(OBJS)

oracle: oracle/build/libstrait_oracle.so

OSRC := $(wildcard oracle/*.c)

oracle/build/libstrait_oracle.so: $(OSRC) $(wildcard include/*.h)
	@mkdir -p oracle/build
	gcc -O2 -fPIC -shared -ffp-contract=off -fno-fast-math -fopenmp -o $@ $(OSRC) -lm

# diagnostic: the replay engine with per-phase cycle accounting (scripts/replay_profile.py)
PROF_LIB := build/prof/_strait.so
PROF_OBJS := $(patsubst $(CDIR)/%.cu,build/prof/%.o,$(CSRC))
prof: $(PROF_LIB)
build/prof/%.o: $(CDIR)/%.cu $(COMMON_HDR) $(REPLAY_HDR)
	@mkdir -p build/prof
	$(NVCC) $(NVFLAGS) -DSTRAIT_REPLAY_PROFILE=1 -dc -o $@ $<
$(PROF_LIB): $(PROF_OBJS)
	$(NVCC) $(ARCH) -shared -Xcompiler -fPIC -o $@ $(PROF_OBJS)

# diagnostic: the sweep with its STRAIT_SWEEP_DIAG timing switches compiled in (scripts/gpu_diag2.sh)
DIAG_LIB := build/diag/_strait.so
DIAG_OBJS := $(patsubst $(CDIR)/%.cu,build/diag/%.o,$(CSRC))
diag: $(DIAG_LIB)
build/diag/%.o: $(CDIR)/%.cu $(COMMON_HDR) $(REPLAY_HDR) $(SWEEP_HDR)
	@mkdir -p build/diag
	$(NVCC) $(NVFLAGS) -DSTRAIT_SWEEP_DIAG_BUILD=1 -dc -o $@ $<
$(DIAG_LIB): $(DIAG_OBJS)
	$(NVCC) $(ARCH) -shared -Xcompiler -fPIC -o $@ $(DIAG_OBJS)

clean:
	rm -rf build $(LIB) oracle/build

.PHONY: all oracle clean prof diag
