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
CHDR := $(wildcard paper_2604_28175_b200/csrc/*.cuh) include/strait.h
OBJS := $(patsubst paper_2604_28175_b200/csrc/%.cu,build/%.o,$(CSRC))

all: $(LIB)

build/%.o: paper_2604_28175_b200/csrc/%.cu $(CHDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -dc -o $@ $<

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -Xcompiler -fPIC -o $@ $(OBJS)

oracle: oracle/build/libstrait_oracle.so

OSRC := $(wildcard oracle/*.c)

oracle/build/libstrait_oracle.so: $(OSRC) $(wildcard include/*.h)
	@mkdir -p oracle/build
	gcc -O2 -fPIC -shared -ffp-contract=off -fno-fast-math -fopenmp -o $@ $(OSRC) -lm

clean:
	rm -rf build $(LIB) oracle/build

.PHONY: all oracle clean
