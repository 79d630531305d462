# Builds every native artefact in-tree (the .so files travel to the GPU box
# with the gpurun snapshot). __graft_entry__.build() runs `make -j`.
NVCC      ?= nvcc
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall
PKG       := paper_2312_13170_b200
CSRC      := $(PKG)/csrc
KSRC      := $(CSRC)/pb_api.cu $(CSRC)/k_umma.cu $(CSRC)/k_split.cu $(CSRC)/k_stats.cu \
             $(CSRC)/k_matvec.cu $(CSRC)/k_simt.cu $(CSRC)/pb_dist.cu $(CSRC)/k_peer.cu \
             $(CSRC)/k_stencil.cu $(CSRC)/k_gramschmidt.cu $(CSRC)/k_gram.cu $(CSRC)/k_covdist.cu
KOBJ      := $(patsubst $(CSRC)/%.cu,build/%.o,$(KSRC))
HDRS      := include/pb.h $(CSRC)/pb_internal.h $(CSRC)/pb_check.h $(CSRC)/pb_device.cuh $(CSRC)/pb_band_prep.cuh $(CSRC)/pb_umma.cuh

all: $(PKG)/libpb.so oracle/libpb_oracle.so pbgen/libpbgen_host.so pbgen/libpbgen_dev.so

build/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -Xptxas -v -c $< -o $@ 2> build/$*.ptxas.txt || (cat build/$*.ptxas.txt; false)

$(PKG)/libpb.so: $(KOBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(KOBJ) -ldl

# The oracle: plain C++, fp64, no FMA contraction, no fast-math (test infrastructure only).
oracle/libpb_oracle.so: oracle/pb_oracle.cpp
	g++ -O2 -std=c++17 -fopenmp -ffp-contract=off -shared -fPIC -Wall -o $@ $<

pbgen/libpbgen_host.so: pbgen/pbgen_host.c pbgen/pbgen_core.h
	gcc -O2 -fopenmp -ffp-contract=off -shared -fPIC -Wall -o $@ $<

pbgen/libpbgen_dev.so: pbgen/pbgen_dev.cu pbgen/pbgen_core.h
	$(NVCC) $(ARCH) -O3 -shared -Xcompiler -fPIC -o $@ $<

clean:
	rm -rf build $(PKG)/libpb.so oracle/libpb_oracle.so pbgen/*.so

.PHONY: all clean
