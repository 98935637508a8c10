# librs_b200.so — the B200-native planning core (sm_100a only).
NVCC     ?= nvcc
ARCH     := -gencode arch=compute_100a,code=sm_100a
PKG      := paper_2602_22718_b200
SRCS     := $(wildcard $(PKG)/csrc/*.cu)
HDRS     := $(wildcard $(PKG)/csrc/*.cuh) include/rs.h include/rs_scenario_tables.h
NVFLAGS  := $(ARCH) -O3 -lineinfo --fmad=false -std=c++17 -Iinclude -Xcompiler -fPIC \
            -Xptxas -v --expt-relaxed-constexpr
LIB      := $(PKG)/librs_b200.so
OBJDIR   := build/obj

.PHONY: all lib oracle ref clean
all: lib oracle

lib: $(LIB)

$(OBJDIR)/%.o: $(PKG)/csrc/%.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -dc $< -o $@ 2> $(OBJDIR)/$*.ptxas.log || (cat $(OBJDIR)/$*.ptxas.log; exit 1)

$(LIB): $(patsubst $(PKG)/csrc/%.cu,$(OBJDIR)/%.o,$(SRCS))
	$(NVCC) $(ARCH) -shared -Xcompiler -fPIC -cudart static -o $@ $^

oracle:
	$(MAKE) -C oracle port

ref:
	$(MAKE) -C oracle ref

clean:
	rm -rf build $(LIB)
