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

.PHONY: all lib oracle ref clean prof
# Phase-timing build (tools/phases.py; RS_B200_LIB selects it): not the product.
PROF_LIB := build/librs_b200_prof.so
prof: $(PROF_LIB)
build/objp/%.o: $(PKG)/csrc/%.cu $(HDRS)
	@mkdir -p build/objp
	$(NVCC) $(NVFLAGS) -DRS_PROFILE_PHASES -dc $< -o $@ 2> build/objp/$*.ptxas.log || (cat build/objp/$*.ptxas.log; exit 1)
$(PROF_LIB): $(patsubst $(PKG)/csrc/%.cu,build/objp/%.o,$(SRCS))
	$(NVCC) $(ARCH) -shared -Xcompiler -fPIC -cudart static -o $@ $^ -ldl

all: lib oracle

lib: $(LIB)

$(OBJDIR)/%.o: $(PKG)/csrc/%.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -dc $< -o $@ 2> $(OBJDIR)/$*.ptxas.log || (cat $(OBJDIR)/$*.ptxas.log; exit 1)

$(LIB): $(patsubst $(PKG)/csrc/%.cu,$(OBJDIR)/%.o,$(SRCS))
	$(NVCC) $(ARCH) -shared -Xcompiler -fPIC -cudart static -o $@ $^ -ldl

oracle:
	$(MAKE) -C oracle port

ref:
	$(MAKE) -C oracle ref

clean:
	rm -rf build $(LIB)

# ---------------------------------------------------------------------------
# C++ drop-in for the reference `rollsim` library (needs /root/reference at
# build time; the outputs travel in build/shim/). librollsim_b200.a = the
# reference's own objects minus dedup.o / planner.o + our shim, which calls
# librs_b200.so. The reference's test suites are relinked against it
# (*_b200) and, to validate the minimal doctest harness, against the
# unmodified reference library (*_ref).
REF       ?= /root/reference/proj
NLOHMANN  ?= /opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty
SHIM_OUT  := build/shim
# the reference's non-hot-path units, compiled for the drop-in under build/shim
# (apart from the oracle build in oracle/_ref), with the reference's flags
REF_OBJ   := $(SHIM_OUT)/ref
REF_KEEP  := workload predictor profile placement simulator training report cli
SHIM_SRCS := $(wildcard $(PKG)/shim/*.cpp)
SHIM_OBJS := $(patsubst $(PKG)/shim/%.cpp,$(SHIM_OUT)/%.o,$(SHIM_SRCS))
CXXREF    := g++ -std=c++20 -O3 -DNDEBUG -Wall -Wextra -fPIC -I$(REF)/include \
             -Ioracle/include_shim -I$(NLOHMANN) -Iinclude
SUITES    := acceptance_main test_dedup test_planner test_profile test_training

.PHONY: shim
shim: $(foreach t,$(SUITES),$(SHIM_OUT)/$(t)_b200 $(SHIM_OUT)/$(t)_ref) \
      $(SHIM_OUT)/test_placement_b200 $(SHIM_OUT)/test_trace_b200 $(SHIM_OUT)/c5_bench_b200 $(SHIM_OUT)/c5_bench_ref \
      $(SHIM_OUT)/c5_bench_train $(SHIM_OUT)/test_training_train $(SHIM_OUT)/test_simulator_train \
      $(SHIM_OUT)/c3_bench_b200 $(SHIM_OUT)/c3_bench_ref

# C3 driver (shim/tools/c3_bench.cpp): scale() at 64K x G=8, N in [1, 512]
$(SHIM_OUT)/c3_bench_b200: $(PKG)/shim/tools/c3_bench.cpp $(SHIM_OUT)/librollsim_b200.a $(LIB)
	$(CXXREF) $< -o $@ $(SHIM_OUT)/librollsim_b200.a -L$(PKG) -lrs_b200 \
	    -Wl,-rpath,'$$ORIGIN/../../$(PKG)' -lpthread

$(SHIM_OUT)/c3_bench_ref: $(PKG)/shim/tools/c3_bench.cpp ref
	@mkdir -p $(SHIM_OUT)
	$(CXXREF) $< -o $@ oracle/_ref/librollsim_ref.a -lpthread

# C5 driver (shim/tools/c5_bench.cpp): the reference's run_training linked three ways
$(SHIM_OUT)/c5_bench_b200: $(PKG)/shim/tools/c5_bench.cpp $(SHIM_OUT)/librollsim_b200.a $(LIB)
	$(CXXREF) $< -o $@ $(SHIM_OUT)/librollsim_b200.a -L$(PKG) -lrs_b200 \
	    -Wl,-rpath,'$$ORIGIN/../../$(PKG)' -lpthread

$(SHIM_OUT)/c5_bench_ref: $(PKG)/shim/tools/c5_bench.cpp ref
	@mkdir -p $(SHIM_OUT)
	$(CXXREF) $< -o $@ oracle/_ref/librollsim_ref.a -lpthread

# INTEGRATION.md's swap as a maintainer applies it: the committed patch on a
# build-time copy of the reference's training.cpp (outputs under build/ only)
$(SHIM_OUT)/training_b200.cpp: $(REF)/src/training.cpp $(PKG)/shim/patches/training_b200.patch
	@mkdir -p $(SHIM_OUT)
	patch -s -o $@ $(REF)/src/training.cpp $(PKG)/shim/patches/training_b200.patch

$(SHIM_OUT)/training_b200.o: $(SHIM_OUT)/training_b200.cpp $(PKG)/shim/rollsim_b200.hpp
	$(CXXREF) -I$(PKG)/shim -c $< -o $@

# and the simulator's dispatch pass skipped while no actor holds a queued cut
# (shim/patches/simulator_b200.patch; run_step's results are unchanged)
$(SHIM_OUT)/simulator_b200.cpp: $(REF)/src/simulator.cpp $(PKG)/shim/patches/simulator_b200.patch
	@mkdir -p $(SHIM_OUT)
	patch -s -o $@ $(REF)/src/simulator.cpp $(PKG)/shim/patches/simulator_b200.patch

$(SHIM_OUT)/simulator_b200.o: $(SHIM_OUT)/simulator_b200.cpp
	$(CXXREF) -c $< -o $@

$(SHIM_OUT)/librollsim_b200_train.a: $(SHIM_OBJS) $(SHIM_OUT)/training_b200.o $(SHIM_OUT)/simulator_b200.o \
    $(addprefix $(REF_OBJ)/,$(addsuffix .o,$(filter-out training simulator,$(REF_KEEP))))
	rm -f $@
	ar rcs $@ $(SHIM_OBJS) $(SHIM_OUT)/training_b200.o $(SHIM_OUT)/simulator_b200.o \
	    $(addprefix $(REF_OBJ)/,$(addsuffix .o,$(filter-out training simulator,$(REF_KEEP))))

$(SHIM_OUT)/c5_bench_train: $(PKG)/shim/tools/c5_bench.cpp $(SHIM_OUT)/librollsim_b200_train.a $(LIB)
	$(CXXREF) $< -o $@ $(SHIM_OUT)/librollsim_b200_train.a -L$(PKG) -lrs_b200 \
	    -Wl,-rpath,'$$ORIGIN/../../$(PKG)' -lpthread

# the reference's own simulator suite against the patched simulator.cpp
$(SHIM_OUT)/test_simulator_train: $(REF)/tests/test_simulator.cpp $(SHIM_OUT)/librollsim_b200_train.a $(LIB)
	$(CXXREF) -I$(PKG)/shim/doctest $< -o $@ $(SHIM_OUT)/librollsim_b200_train.a \
	    -L$(PKG) -lrs_b200 -Wl,-rpath,'$$ORIGIN/../../$(PKG)' -lpthread

# the reference's own training suite against the patched training.cpp
$(SHIM_OUT)/test_training_train: $(REF)/tests/test_training.cpp $(SHIM_OUT)/librollsim_b200_train.a $(LIB)
	$(CXXREF) -I$(PKG)/shim/doctest $< -o $@ $(SHIM_OUT)/librollsim_b200_train.a \
	    -L$(PKG) -lrs_b200 -Wl,-rpath,'$$ORIGIN/../../$(PKG)' -lpthread

# drop-in extension suite (rollsim_b200.hpp) against the stock penalty path
$(SHIM_OUT)/test_placement_b200: $(PKG)/shim/tests/test_placement_b200.cpp $(SHIM_OUT)/librollsim_b200.a $(LIB)
	$(CXXREF) -I$(PKG)/shim -I$(PKG)/shim/doctest $< -o $@ $(SHIM_OUT)/librollsim_b200.a \
	    -L$(PKG) -lrs_b200 -Wl,-rpath,'$$ORIGIN/../../$(PKG)' -lpthread

$(SHIM_OUT)/test_trace_b200: $(PKG)/shim/tests/test_trace_b200.cpp $(SHIM_OUT)/librollsim_b200.a $(LIB)
	$(CXXREF) -I$(PKG)/shim -I$(PKG)/shim/doctest $< -o $@ $(SHIM_OUT)/librollsim_b200.a \
	    -L$(PKG) -lrs_b200 -Wl,-rpath,'$$ORIGIN/../../$(PKG)' -lpthread

$(REF_OBJ)/%.o: $(REF)/src/%.cpp
	@mkdir -p $(REF_OBJ)
	$(CXXREF) -c $< -o $@

$(SHIM_OUT)/%.o: $(PKG)/shim/%.cpp $(PKG)/shim/rs_shim.hpp $(PKG)/shim/rollsim_b200.hpp include/rs.h
	@mkdir -p $(SHIM_OUT)
	$(CXXREF) -c $< -o $@

$(SHIM_OUT)/librollsim_b200.a: $(SHIM_OBJS) $(addprefix $(REF_OBJ)/,$(addsuffix .o,$(REF_KEEP)))
	rm -f $@
	ar rcs $@ $(SHIM_OBJS) $(addprefix $(REF_OBJ)/,$(addsuffix .o,$(REF_KEEP)))

$(SHIM_OUT)/%_b200: $(REF)/tests/%.cpp $(SHIM_OUT)/librollsim_b200.a $(LIB)
	$(CXXREF) -I$(PKG)/shim/doctest $< -o $@ $(SHIM_OUT)/librollsim_b200.a \
	    -L$(PKG) -lrs_b200 -Wl,-rpath,'$$ORIGIN/../../$(PKG)' -lpthread

$(SHIM_OUT)/%_ref: $(REF)/tests/%.cpp ref
	@mkdir -p $(SHIM_OUT)
	$(CXXREF) -I$(PKG)/shim/doctest $< -o $@ oracle/_ref/librollsim_ref.a -lpthread
