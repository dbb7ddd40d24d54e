#!/bin/bash
# Compile A/B variants of libpropring.so (preprocessor knobs in csrc/*.cu) into _variants/ for profiling:
#   tools/variants.sh NAME "-DKNOB=V ..."  ->  _variants/libpropring_NAME.so  (load with PROPRING_LIB=...)
set -e
cd "$(dirname "$0")/.."
name=$1; shift
out=_variants/$name; mkdir -p $out
NVCC="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC,-ffp-contract=off -I include $*"
for f in shard gather ring update; do $NVCC -c paper_2111_08272_b200/csrc/$f.cu -o $out/$f.o; done
g++ -O2 -std=c++17 -fPIC -ffp-contract=off -I include -c paper_2111_08272_b200/csrc/alloc.cpp -o $out/alloc.o
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o _variants/libpropring_$name.so $out/*.o
echo _variants/libpropring_$name.so
