#!/usr/bin/env bash
# Builds build/prof/libgpk.so with the SGD slab's per-role wait instrumentation
# (-DSGD_PROF=1; development only), from the normal build's other objects.
set -e
cd "$(dirname "$0")/../paper_2405_18457_b200"
make -s -j8
mkdir -p build/prof
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -DSGD_PROF=1 \
  -Xcompiler -fPIC,-O3,-ffp-contract=off --expt-relaxed-constexpr -c csrc/sgd_lazy.cu -o build/prof/sgd_lazy.o
objs=$(ls build/*.o | grep -v sgd_lazy.o)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/prof/libgpk.so build/prof/sgd_lazy.o $objs \
  -L/usr/local/cuda/lib64 -lcublas -lcusolver -ldl -Xlinker -rpath,/usr/local/cuda/lib64
