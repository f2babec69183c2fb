#!/usr/bin/env bash
# Development: builds build/<name>/libgpk.so with extra nvcc defines for the SGD
# slab (timing experiments; e.g. SGD_FAKE_DIST=1 / SGD_FAKE_MUFU=1 drop work and
# give wrong results). usage: tools/sgd_variant_build.sh <name> -DSGD_FAKE_DIST=1 ...
set -e
name=$1; shift
cd "$(dirname "$0")/../paper_2405_18457_b200"
make -s -j8
mkdir -p build/$name
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 "$@" \
  -Xcompiler -fPIC,-O3,-ffp-contract=off --expt-relaxed-constexpr -c csrc/sgd_lazy.cu -o build/$name/sgd_lazy.o
objs=$(ls build/*.o | grep -v sgd_lazy.o)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/$name/libgpk.so build/$name/sgd_lazy.o $objs \
  -L/usr/local/cuda/lib64 -lcublas -lcusolver -ldl -Xlinker -rpath,/usr/local/cuda/lib64
