#!/bin/bash
# Build a variant of libisoclust_b200.so with one source recompiled under
# extra defines:  tools/build_variant.sh NAME SOURCE.cu "-DFOO=1 ..."
# -> variants/NAME.so (git-ignored; travels with gpurun like the main .so)
set -e
name=$1; src=$2; defs=$3
cd "$(dirname "$0")/../paper_1702_04739_b200/csrc"
make -s
out=../../variants/$name; mkdir -p $out
base=$(basename $src .cu)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -O2 \
     -Xptxas -v --expt-relaxed-constexpr -cudart static -fmad=false $defs -dc -o $out/$base.o $src 2> $out/ptxas.log \
     || (cat $out/ptxas.log; false)
objs=$(ls build/*.o | grep -v "build/$base.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o ../../variants/$name.so $objs $out/$base.o
grep -A2 "Function properties for .*sym_kernel" $out/ptxas.log | grep -v Compiling || true
