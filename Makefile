# Builds paper_2209_06916_b200/_lib/libmgrit_b200.so for sm_100a (B200).
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 -Xptxas -v --expt-relaxed-constexpr
SRC := paper_2209_06916_b200/csrc
OUT := paper_2209_06916_b200/_lib
BUILD := build/obj
OBJS := $(BUILD)/mgb_host.o $(BUILD)/k_win_exact.o $(BUILD)/k_win_fast.o $(BUILD)/k_gen.o $(BUILD)/k_rk.o $(BUILD)/k_slgc.o $(BUILD)/k_slgc1.o
HDRS := $(SRC)/mgb_device.cuh $(SRC)/mgb_cluster.cuh $(SRC)/mgb_cluster1.cuh $(SRC)/mgb_registry.h include/mgrit_b200.h

all: $(OUT)/libmgrit_b200.so

$(BUILD)/%.o: $(SRC)/%.cu $(HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -c $< -o $@ > $(BUILD)/$*.ptxas.log 2>&1 || (cat $(BUILD)/$*.ptxas.log; exit 1)

$(OUT)/libmgrit_b200.so: $(OBJS)
	@mkdir -p $(OUT)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS)

clean:
	rm -rf build $(OUT)/libmgrit_b200.so

.PHONY: all clean

# phase-timer build of the cluster kernel (tools/cluster_trace.py; not shipped)
TRACE_BUILD := build/trace
$(TRACE_BUILD)/%.o: $(SRC)/%.cu $(HDRS)
	@mkdir -p $(TRACE_BUILD)
	$(NVCC) $(NVFLAGS) -DMGB_CL_TRACE -c $< -o $@ > $(TRACE_BUILD)/$*.log 2>&1 || (cat $(TRACE_BUILD)/$*.log; exit 1)
trace: $(patsubst $(BUILD)/%,$(TRACE_BUILD)/%,$(OBJS))
	$(NVCC) $(ARCH) -shared -o $(OUT)/libmgrit_b200_trace.so $^
.PHONY: trace
