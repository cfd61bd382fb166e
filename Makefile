# Builds the in-tree C-ABI library (travels to the GPU box with the snapshot).
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -Xptxas -v
SRC := paper_2103_07706_b200/csrc
LIB := paper_2103_07706_b200/lib/libpswe_b200.so
HDRS := $(wildcard $(SRC)/*.cuh) include/pswe_b200.h

all: $(LIB)

$(LIB): $(SRC)/pswe_capi.cu $(HDRS)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRC)/pswe_capi.cu 2> paper_2103_07706_b200/lib/ptxas.log || (cat paper_2103_07706_b200/lib/ptxas.log; false)

clean:
	rm -f $(LIB)

.PHONY: all clean
