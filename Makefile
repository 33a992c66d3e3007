# Builds the B200 CudaDnn C-ABI library and the C++ host libraries in-tree.
#   make -j8            everything (nvcc cross-compiles sm_100a without a GPU)
NVCC     ?= nvcc
CXX      ?= g++
ARCH     := -gencode arch=compute_100a,code=sm_100a
NVFLAGS  := -std=c++20 $(ARCH) -O3 -lineinfo -Xcompiler -fPIC,-fvisibility=hidden -Iinclude \
            --expt-relaxed-constexpr -Xptxas -warn-spills
CXXFLAGS := -std=c++20 -O3 -fPIC -Wall -Wextra -Iinclude
PKG      := paper_1810_02272_b200
LIB      := $(PKG)/lib
OBJ      := build/obj
CU_SRC   := $(wildcard $(PKG)/csrc/cudadnn/*.cu)
CU_HDR   := $(wildcard $(PKG)/csrc/cudadnn/*.cuh $(PKG)/csrc/cudadnn/*.hpp) include/cudadnn.h
CU_OBJ   := $(patsubst $(PKG)/csrc/cudadnn/%.cu,$(OBJ)/cudadnn/%.o,$(CU_SRC))
CUDA_LIB := $(dir $(shell which $(NVCC)))../lib64

PG_SRC   := $(wildcard $(PKG)/csrc/polegrad/*.cpp)
PG_HDR   := $(wildcard include/polegrad/*.hpp $(PKG)/csrc/polegrad/*.hpp)
PG_OBJ32 := $(patsubst $(PKG)/csrc/polegrad/%.cpp,$(OBJ)/pg32/%.o,$(PG_SRC))
PG_OBJ64 := $(patsubst $(PKG)/csrc/polegrad/%.cpp,$(OBJ)/pg64/%.o,$(PG_SRC))

all: $(LIB)/libcudadnn.so $(LIB)/libpolegrad_b200_f32.so $(LIB)/libpolegrad_b200_f64.so

$(OBJ)/cudadnn/%.o: $(PKG)/csrc/cudadnn/%.cu $(CU_HDR)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB)/libcudadnn.so: $(CU_OBJ)
	@mkdir -p $(LIB)
	$(NVCC) $(ARCH) -shared -o $@ $^ -L$(CUDA_LIB) -lcudart_static -ldl -lpthread -lrt \
	  -Xlinker -soname=libcudadnn.so

$(OBJ)/pg32/%.o: $(PKG)/csrc/polegrad/%.cpp $(PG_HDR) include/cudadnn.h
	@mkdir -p $(dir $@)
	$(CXX) $(CXXFLAGS) -DPOLEGRAD_SINGLE_PRECISION -c $< -o $@

$(OBJ)/pg64/%.o: $(PKG)/csrc/polegrad/%.cpp $(PG_HDR) include/cudadnn.h
	@mkdir -p $(dir $@)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(LIB)/libpolegrad_b200_f32.so: $(PG_OBJ32) $(LIB)/libcudadnn.so
	$(CXX) -shared -o $@ $(PG_OBJ32) -L$(LIB) -lcudadnn -Wl,-rpath,'$$ORIGIN'

$(LIB)/libpolegrad_b200_f64.so: $(PG_OBJ64) $(LIB)/libcudadnn.so
	$(CXX) -shared -o $@ $(PG_OBJ64) -L$(LIB) -lcudadnn -Wl,-rpath,'$$ORIGIN'

clean:
	rm -rf build $(LIB)

.PHONY: all clean
