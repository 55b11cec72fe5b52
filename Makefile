# Top-level build (invoked by __graft_entry__.build()).
#
#   paper_2210_04847_b200/lib/libvoxmarch_b200.so  — CUDA kernels + C ABI (sm_100a)
#   paper_2210_04847_b200/lib/libvoxmarch_cpp.so   — C++ drop-in facade (namespace voxmarch)
#   build/vm_cpp_tests                              — C++ facade tests (run under pytest -m gpu)
#   oracle/_build, oracle/_ref                      — CPU oracle (test infrastructure)
#
# The decision path is compiled with --fmad=false (and the host side with
# -ffp-contract=off) so every fp64 expression rounds exactly like the reference.
NVCC     ?= /usr/local/cuda/bin/nvcc
CXX      ?= g++
ARCH     := -gencode arch=compute_100a,code=sm_100a
PKG      := paper_2210_04847_b200
SRC      := $(PKG)/csrc
LIB      := $(PKG)/lib
NVFLAGS  := $(ARCH) -O3 -lineinfo -std=c++17 --fmad=false -Xcompiler -fPIC \
            -Xcompiler -ffp-contract=off -Xptxas -v -Iinclude
CU_SRCS  := $(SRC)/runtime.cu $(SRC)/scan.cu $(SRC)/grid.cu $(SRC)/march.cu $(SRC)/render.cu $(SRC)/camera.cu $(SRC)/voxfield.cu $(SRC)/train.cu $(SRC)/ops.cu $(SRC)/sort.cu
CU_OBJS  := $(patsubst $(SRC)/%.cu,build/obj/%.o,$(CU_SRCS))
HDRS     := $(SRC)/vm_internal.h $(SRC)/vm_exact.cuh $(SRC)/vm_scan.cuh $(SRC)/vm_bulk.cuh include/vmb200.h include/vmb200_types.h

CXXFLAGS := -std=c++20 -O2 -fPIC -ffp-contract=off -Wall -Wextra -Iinclude -I$(SRC)

.PHONY: all oracle ref_unit clean
all: $(LIB)/libvoxmarch_b200.so $(LIB)/libvoxmarch_cpp.so build/vm_cpp_tests oracle ref_unit

# the reference's own unit tests compiled against the facade (tests/ref_unit/Makefile)
ref_unit: $(LIB)/libvoxmarch_cpp.so
	$(MAKE) -f tests/ref_unit/Makefile

# C++ drop-in facade (namespace voxmarch) over the C ABI
$(LIB)/libvoxmarch_cpp.so: $(SRC)/facade.cpp include/voxmarch/voxmarch.hpp $(HDRS) $(LIB)/libvoxmarch_b200.so
	$(CXX) $(CXXFLAGS) -shared -o $@ $(SRC)/facade.cpp -L$(LIB) -lvoxmarch_b200 -Wl,-rpath,'$$ORIGIN'

# C++ facade tests (run on a GPU by tests/test_cpp_facade.py)
build/vm_cpp_tests: tests/cpp/test_facade.cpp tests/cpp/mini_check.hpp include/voxmarch/voxmarch.hpp $(LIB)/libvoxmarch_cpp.so
	@mkdir -p build
	$(CXX) $(CXXFLAGS) -o $@ tests/cpp/test_facade.cpp -L$(LIB) -lvoxmarch_cpp -lvoxmarch_b200 \
	    -Wl,-rpath,'$$ORIGIN/../$(LIB)'

build/obj/%.o: $(SRC)/%.cu $(HDRS)
	@mkdir -p build/obj
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/obj/$*.ptxas.log || (cat build/obj/$*.ptxas.log; false)

build/obj/comm.o: $(SRC)/comm.cpp $(HDRS)
	@mkdir -p build/obj
	$(NVCC) $(NVFLAGS) -x cu -c $< -o $@ 2> build/obj/comm.ptxas.log || (cat build/obj/comm.ptxas.log; false)

$(LIB)/libvoxmarch_b200.so: $(CU_OBJS) build/obj/comm.o
	@mkdir -p $(LIB)
	$(NVCC) $(ARCH) -shared -o $@ $^ -cudart static -ldl -lpthread

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(LIB)
	$(MAKE) -C oracle clean

# A/B variants (experiments): make variant DEFS="-DVMB_WALK_MINB=4" NAME=minb4
variant:
	@mkdir -p build/var_$(NAME) $(LIB)/variants
	for f in $(CU_SRCS); do b=$$(basename $$f .cu); $(NVCC) $(NVFLAGS) $(DEFS) -c $$f -o build/var_$(NAME)/$$b.o 2> build/var_$(NAME)/$$b.log || exit 1; done
	$(NVCC) $(NVFLAGS) $(DEFS) -x cu -c $(SRC)/comm.cpp -o build/var_$(NAME)/comm.o 2> /dev/null
	$(NVCC) $(ARCH) -shared -o $(LIB)/variants/libvoxmarch_b200_$(NAME).so build/var_$(NAME)/*.o -cudart static -ldl -lpthread
