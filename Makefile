# Builds the in-tree sm_100a library paper_2501_07145_b200/_lib/libsigkern_b200.so.
# cudart is linked statically so the .so loads (symbol check) without a GPU.
NVCC      ?= nvcc
ARCH      ?= -gencode arch=compute_100a,code=sm_100a
NVFLAGS   ?= -O3 -lineinfo -std=c++17 $(ARCH) -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
             --expt-relaxed-constexpr -Xptxas -v
SRC_DIR   := paper_2501_07145_b200/csrc
OUT_DIR   := paper_2501_07145_b200/_lib
OBJ_DIR   := build/obj
LIB       := $(OUT_DIR)/libsigkern_b200.so
SRCS      := $(wildcard $(SRC_DIR)/*.cu)
OBJS      := $(patsubst $(SRC_DIR)/%.cu,$(OBJ_DIR)/%.o,$(SRCS))
HDRS      := $(wildcard $(SRC_DIR)/*.cuh) include/sigkern_b200.h

.PHONY: all clean
all: $(LIB)

$(OBJ_DIR)/%.o: $(SRC_DIR)/%.cu $(HDRS)
	@mkdir -p $(OBJ_DIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(OBJ_DIR)/$*.ptxas.log || (cat $(OBJ_DIR)/$*.ptxas.log; false)

$(LIB): $(OBJS)
	@mkdir -p $(OUT_DIR)
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $(OBJS) -Xcompiler -fvisibility=hidden

clean:
	rm -rf build $(LIB)
