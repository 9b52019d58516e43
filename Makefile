# Build for B200 (sm_100a) only. `make` builds the product libraries in-tree
# (they travel to the GPU box with the gpurun snapshot) plus the test-only
# oracle and probe programs.

NVCC     ?= /usr/local/cuda/bin/nvcc
CXX      ?= g++
ARCH     := -gencode arch=compute_100a,code=sm_100a
PKG      := paper_2103_04930_b200
CUDA_DIR := $(PKG)/csrc/cuda
HOST_DIR := $(PKG)/csrc/host
LIB      := $(PKG)/lib
BIN      := $(PKG)/bin
NVFLAGS  := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall --expt-relaxed-constexpr
CXXFLAGS := -std=c++20 -O2 -fPIC -Wall -Wextra -I/usr/local/cuda/include -Iinclude

CUDA_SRCS := $(wildcard $(CUDA_DIR)/*.cu) $(wildcard $(CUDA_DIR)/*.cpp)
CUDA_HDRS := $(wildcard $(CUDA_DIR)/*.hpp) $(wildcard $(CUDA_DIR)/*.cuh) include/avec_cuda.h
CUDA_OBJS := $(patsubst $(CUDA_DIR)/%,build/obj/cuda/%.o,$(CUDA_SRCS))

HOST_SRCS := $(filter-out $(HOST_DIR)/%_main.cpp,$(wildcard $(HOST_DIR)/*.cpp))
HOST_HDRS := $(wildcard $(HOST_DIR)/*.hpp) include/avec_cuda.h
HOST_OBJS := $(patsubst $(HOST_DIR)/%.cpp,build/obj/host/%.o,$(HOST_SRCS))

.PHONY: all product oracle probe clean tsan asan
all: product oracle probe

product: $(LIB)/libavec_cuda.so $(LIB)/libavec_host.so $(BIN)/avec-server $(BIN)/avec-loadgen

build/obj/cuda/%.cu.o: $(CUDA_DIR)/%.cu $(CUDA_HDRS)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -c $< -o $@

build/obj/cuda/%.cpp.o: $(CUDA_DIR)/%.cpp $(CUDA_HDRS)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -x cu -c $< -o $@

$(LIB)/libavec_cuda.so: $(CUDA_OBJS)
	@mkdir -p $(LIB)
	$(NVCC) $(ARCH) -shared -o $@ $^ -lcudart_static -ldl -lpthread -lrt

build/obj/host/%.o: $(HOST_DIR)/%.cpp $(HOST_HDRS)
	@mkdir -p $(dir $@)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(LIB)/libavec_host.so: $(HOST_OBJS) $(LIB)/libavec_cuda.so
	$(CXX) -shared -o $@ $(HOST_OBJS) -L$(LIB) -lavec_cuda -Wl,-rpath,'$$ORIGIN' -l:libcrypto.a -lpthread

$(BIN)/avec-server: $(HOST_DIR)/server_main.cpp $(LIB)/libavec_host.so
	@mkdir -p $(BIN)
	$(CXX) $(CXXFLAGS) -o $@ $< -L$(LIB) -lavec_host -lavec_cuda -Wl,-rpath,'$$ORIGIN/../lib' -lpthread

$(BIN)/avec-loadgen: $(HOST_DIR)/loadgen_main.cpp $(LIB)/libavec_host.so
	@mkdir -p $(BIN)
	$(CXX) $(CXXFLAGS) -o $@ $< -L$(LIB) -lavec_host -lavec_cuda -Wl,-rpath,'$$ORIGIN/../lib' -lpthread

# test-only: the same server over a CPU stub backend (tests/native), for
# protocol tests without a GPU
build/avec_stub_server: tests/native/stub_server.cpp $(LIB)/libavec_host.so
	@mkdir -p build
	$(CXX) $(CXXFLAGS) -I$(HOST_DIR) -o $@ $< -L$(LIB) -lavec_host -lavec_cuda -Wl,-rpath,'$$ORIGIN/../$(LIB)' -lpthread

# the reference drivers include ref_b200_server, which links libavec_cuda.so
oracle: $(LIB)/libavec_cuda.so
	$(MAKE) -C oracle oracle
	@if [ -d /root/reference/proj ]; then $(MAKE) -C oracle ref; else echo "no /root/reference: using prebuilt oracle/_ref"; fi

# ThreadSanitizer build of the host server (libavec_host sources + the CPU
# stub backend) for the protocol tests: AVEC_STUB_BIN=build/tsan/avec_stub_server
TSAN_CXX ?= /usr/bin/g++
TSAN_FLAGS := -std=c++20 -O1 -g -fsanitize=thread -fPIC -I/usr/local/cuda/include -Iinclude
build/tsan/avec_stub_server: tests/native/stub_server.cpp $(HOST_SRCS) $(HOST_HDRS) $(LIB)/libavec_cuda.so
	@mkdir -p build/tsan
	$(TSAN_CXX) $(TSAN_FLAGS) -I$(HOST_DIR) -o $@ tests/native/stub_server.cpp $(HOST_SRCS) -L$(LIB) -lavec_cuda \
	  -Wl,-rpath,'$$ORIGIN/../../$(LIB)' -l:libcrypto.a -lpthread
tsan: build/tsan/avec_stub_server

# AddressSanitizer + UBSan build of the same (AVEC_STUB_BIN=build/asan/avec_stub_server)
ASAN_FLAGS := -std=c++20 -O1 -g -fsanitize=address,undefined -fno-omit-frame-pointer -fPIC -I/usr/local/cuda/include -Iinclude
build/asan/avec_stub_server: tests/native/stub_server.cpp $(HOST_SRCS) $(HOST_HDRS) $(LIB)/libavec_cuda.so
	@mkdir -p build/asan
	$(TSAN_CXX) $(ASAN_FLAGS) -I$(HOST_DIR) -o $@ tests/native/stub_server.cpp $(HOST_SRCS) -L$(LIB) -lavec_cuda \
	  -Wl,-rpath,'$$ORIGIN/../../$(LIB)' -l:libcrypto.a -lpthread
asan: build/asan/avec_stub_server

probe: build/tc_probe build/tc2_probe build/tma3d_probe
build/tc_probe: tests/native/tc_probe.cu $(CUDA_DIR)/ptx.cuh
	@mkdir -p build
	$(NVCC) $(ARCH) -O3 -lineinfo -std=c++17 -o $@ $<
build/tc2_probe: tests/native/tc2_probe.cu $(CUDA_DIR)/ptx.cuh
	@mkdir -p build
	$(NVCC) $(ARCH) -O3 -lineinfo -std=c++17 -o $@ $<
build/tma3d_probe: tests/native/tma3d_probe.cu $(CUDA_DIR)/ptx.cuh
	@mkdir -p build
	$(NVCC) $(ARCH) -O3 -lineinfo -std=c++17 -o $@ $<

clean:
	rm -rf build $(LIB) $(BIN)
