# Build of the B200 library (sm_100a) and the test-only checkers.
#   make            -> paper_1306_4627_b200/_lib/libwavelcs_b200.so + oracle/
# nvcc cross-compiles here (no GPU needed).
NVCC ?= /usr/local/cuda/bin/nvcc
CXX ?= g++
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Iinclude -Xcompiler -fPIC -Xcompiler -Wall
SRC := paper_1306_4627_b200/csrc
OBJ := build/obj
LIB := paper_1306_4627_b200/_lib/libwavelcs_b200.so
FACADE_TEST := tests/cpp/test_facade
CLI := paper_1306_4627_b200/_lib/wavelcs_b200
CU_SRCS := $(wildcard $(SRC)/*.cu)
CXX_SRCS := $(wildcard $(SRC)/*.cpp)
OBJS := $(patsubst $(SRC)/%.cu,$(OBJ)/%.o,$(CU_SRCS)) $(patsubst $(SRC)/%.cpp,$(OBJ)/%.cpp.o,$(CXX_SRCS))
HDRS := $(wildcard $(SRC)/*.cuh) $(wildcard $(SRC)/*.h) $(wildcard include/*.h) $(wildcard include/*.hpp) $(wildcard include/wavelcs/*.hpp)

all: lib oracle $(FACADE_TEST) $(CLI) reftests

lib: $(LIB)

$(SRC)/rowstep.cuh: $(SRC)/gen_rowstep.py
	python3 $< > $@

$(OBJ)/%.o: $(SRC)/%.cu $(HDRS) $(SRC)/rowstep.cuh
	@mkdir -p $(OBJ)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(OBJ)/%.cpp.o: $(SRC)/%.cpp $(HDRS)
	@mkdir -p $(OBJ)
	$(CXX) -std=c++20 -O2 -fPIC -Wall -Wextra -Iinclude -c $< -o $@

# C++ facade test (the reference's unit cases against wavelcs_b200.hpp);
# lives in tests/ so it travels to the GPU box with the snapshot.
$(FACADE_TEST): tests/cpp/test_facade.cpp $(LIB) include/wavelcs_b200.hpp
	$(CXX) -std=c++20 -O2 -Wall -Wextra -Iinclude -o $@ $< -L$(dir $(LIB)) -lwavelcs_b200 \
	    -Wl,-rpath,'$$ORIGIN/../../$(dir $(LIB))'

# Command-line front end on the GPU path (tools/cli).
$(CLI): tools/cli/wavelcs_b200_main.cpp $(LIB) include/wavelcs_b200.hpp
	$(CXX) -std=c++20 -O2 -Wall -Wextra -Iinclude -o $@ $< -L$(dir $(LIB)) -lwavelcs_b200 \
	    -Wl,-rpath,'$$ORIGIN'

$(LIB): $(OBJS)
	@mkdir -p $(dir $@)
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $^ -lpthread -ldl -lrt

oracle:
	$(MAKE) -s -C oracle

# the reference's unit tests and acceptance suite, compiled unchanged against
# include/wavelcs/ (only where /root/reference exists; prebuilt elsewhere)
reftests: $(LIB) $(CLI)
	$(MAKE) -s -C tests/cpp

clean:
	rm -rf build $(LIB) $(FACADE_TEST) $(CLI)

.PHONY: all lib oracle reftests clean
