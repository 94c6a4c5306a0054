# Builds libspx.so (all sm_100a kernels + the C-ABI in include/spx.h) in-tree, and the
# oracle's C helpers.  `python -c "import __graft_entry__ as g; g.build()"` drives this.
NVCC ?= nvcc
CSRC := paper_2502_19913_b200/csrc
OUT := paper_2502_19913_b200/libspx.so
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -shared --expt-relaxed-constexpr \
           -Xptxas -warn-spills -Iinclude
SRCS := $(wildcard $(CSRC)/*.cu)
HDRS := $(wildcard $(CSRC)/*.cuh) $(wildcard $(CSRC)/*.h) include/spx.h

SCHED := paper_2502_19913_b200/libspx_sched.so

all: $(OUT) $(SCHED)

sched: $(SCHED)

# native path planner (host C++, no CUDA; include/spx_sched.h)
$(SCHED): paper_2502_19913_b200/native_sched/sched.cpp include/spx_sched.h
	$(CXX) -O2 -std=c++17 -ffp-contract=off -fPIC -shared -o $@ $<

$(OUT): $(SRCS) $(HDRS)
	$(NVCC) $(NVFLAGS) -o $@ $(SRCS) -lcudart

ptxas-info: $(SRCS) $(HDRS)
	$(NVCC) $(NVFLAGS) -Xptxas -v -o /tmp/spx_ptxas.so $(SRCS) -lcudart

clean:
	rm -f $(OUT) $(SCHED)

.PHONY: all clean ptxas-info sched
