# Builds the sm_100a C-ABI library in-tree (travels to the GPU box with gpurun)
# and the oracle's optional reference build.  `python -c "import __graft_entry__ as g; g.build()"`
# drives the same targets.
NVCC      ?= nvcc
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr
SRC_DIR   := paper_1306_3277_b200/csrc
LIB_DIR   := paper_1306_3277_b200/lib
SRCS      := $(wildcard $(SRC_DIR)/*.cu)
OBJS      := $(patsubst $(SRC_DIR)/%.cu,build/%.o,$(SRCS))
LIB       := $(LIB_DIR)/libssm_b200.so

all: $(LIB)

build/%.o: $(SRC_DIR)/%.cu $(wildcard $(SRC_DIR)/*.cuh) include/ssm_b200.h
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(LIB): $(OBJS)
	@mkdir -p $(LIB_DIR)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcudart -lnvrtc

clean:
	rm -rf build $(LIB)

.PHONY: all clean
