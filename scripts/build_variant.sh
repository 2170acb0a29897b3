#!/bin/bash
# Build a variant libgc with extra -D flags into build_var/<name>/libgc.so (A/B timing via GC_LIB_PATH).
# usage: scripts/build_variant.sh NAME -DFOO=1 ...
set -e
name=$1; shift
out=build_var/$name; mkdir -p $out
NV="/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr -Iinclude $*"
objs=""
for f in gc_api build_csr tc peel listing comm; do
  $NV -c paper_1708_06866_b200/csrc/$f.cu -o $out/$f.o & objs="$objs $out/$f.o"
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $out/libgc.so $objs -ldl -lpthread -lrt
echo built $out/libgc.so
