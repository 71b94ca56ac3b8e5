# Builds every native artefact in-tree (the .so files travel to the GPU box with
# the gpurun snapshot; they are git-ignored).
#   gen/libqrgen_host.so   host generators (gcc, OpenMP)          — harness, shared by both sides
#   gen/libqrgen_dev.so    device generators (nvcc, sm_100a)      — harness
#   oracle/liboracle.so    CPU oracle (plain C, gcc)              — test infrastructure only
#   paper_2602_04103_b200/lib/libqrank.so   the product C-ABI library (nvcc, sm_100a)
#   examples/qrank_demo    plain-C user of the C ABI (gcc -std=c99, links libqrank.so only)
NVCC    ?= /usr/local/cuda/bin/nvcc
HOSTCC  := gcc
ARCH    := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -lineinfo $(ARCH) -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
           -Xptxas -v --expt-relaxed-constexpr -Iinclude $(QR_EXTRA)
CFLAGS  := -O2 -fPIC -fopenmp -std=c11 -Wall -Wno-unused-function

PKG     := paper_2602_04103_b200
QR_SRC  := $(wildcard $(PKG)/csrc/*.cu)
QR_HDR  := $(wildcard $(PKG)/csrc/*.cuh) include/qrank.h
BUILD   ?= build
QR_OBJ  := $(patsubst $(PKG)/csrc/%.cu,$(BUILD)/qr_%.o,$(QR_SRC))

all: gen/libqrgen_host.so gen/libqrgen_dev.so oracle/liboracle.so $(if $(QR_SRC),$(PKG)/lib/libqrank.so examples/qrank_demo)

gen/libqrgen_host.so: gen/qrgen_host.c gen/qrgen.h
	$(HOSTCC) $(CFLAGS) -shared -o $@ gen/qrgen_host.c

gen/libqrgen_dev.so: gen/qrgen_dev.cu gen/qrgen.h
	$(NVCC) -O3 $(ARCH) -std=c++17 -Xcompiler -fPIC -shared -o $@ gen/qrgen_dev.cu

oracle/liboracle.so: oracle/oracle.c
	$(HOSTCC) $(CFLAGS) -shared -o $@ oracle/oracle.c

$(BUILD)/qr_%.o: $(PKG)/csrc/%.cu $(QR_HDR)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> $(BUILD)/qr_$*.ptxas.txt || (cat $(BUILD)/qr_$*.ptxas.txt; false)

$(PKG)/lib/libqrank.so: $(QR_OBJ)
	@mkdir -p $(PKG)/lib
	$(NVCC) $(ARCH) -shared -o $@ $(QR_OBJ)

examples/qrank_demo: examples/qrank_demo.c include/qrank.h $(PKG)/lib/libqrank.so
	$(HOSTCC) -O2 -std=c99 -Wall -Wextra -pedantic -Iinclude -o $@ examples/qrank_demo.c \
	  -L$(PKG)/lib -lqrank -Wl,-rpath,'$$ORIGIN/../$(PKG)/lib'

clean:
	rm -rf build gen/*.so oracle/*.so $(PKG)/lib/*.so examples/qrank_demo

.PHONY: all clean
