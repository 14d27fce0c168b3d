# Build of the B200 library (sm_100a) and the test-only checkers.
#   make            -> paper_1306_4627_b200/_lib/libwavelcs_b200.so + oracle/
# nvcc cross-compiles here (no GPU needed).
NVCC ?= /usr/local/cuda/bin/nvcc
CXX ?= g++
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall
SRC := paper_1306_4627_b200/csrc
OBJ := build/obj
LIB := paper_1306_4627_b200/_lib/libwavelcs_b200.so
CU_SRCS := $(wildcard $(SRC)/*.cu)
CXX_SRCS := $(wildcard $(SRC)/*.cpp)
OBJS := $(patsubst $(SRC)/%.cu,$(OBJ)/%.o,$(CU_SRCS)) $(patsubst $(SRC)/%.cpp,$(OBJ)/%.cpp.o,$(CXX_SRCS))
HDRS := $(wildcard $(SRC)/*.cuh) $(wildcard $(SRC)/*.h) $(wildcard include/*.h) $(wildcard include/*.hpp)

all: lib oracle

lib: $(LIB)

$(SRC)/rowstep.cuh: $(SRC)/gen_rowstep.py
	python3 $< > $@

$(OBJ)/%.o: $(SRC)/%.cu $(HDRS) $(SRC)/rowstep.cuh
	@mkdir -p $(OBJ)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(OBJ)/%.cpp.o: $(SRC)/%.cpp $(HDRS)
	@mkdir -p $(OBJ)
	$(CXX) -std=c++17 -O2 -fPIC -Wall -Wextra -Iinclude -c $< -o $@

$(LIB): $(OBJS)
	@mkdir -p $(dir $@)
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $^ -lpthread -ldl -lrt

oracle:
	$(MAKE) -s -C oracle

clean:
	rm -rf build $(LIB)

.PHONY: all lib oracle clean
