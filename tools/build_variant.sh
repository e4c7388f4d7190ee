#!/bin/bash
# Build an engine variant with extra nvcc defines into build/variants/NAME/
#   tools/build_variant.sh NAME [-DMACRO=V ...]   (bench it with tools/varbench.sh)
set -e
name=$1; shift
d=build/variants/$name
mkdir -p $d
make -s lib >/dev/null
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo -fmad=false \
  -ccbin /usr/bin/g++ -Xcompiler -fPIC -Xptxas -v -Iinclude "$@" \
  -c paper_2108_03076_b200/csrc/mc_engine.cu -o $d/mc_engine.o 2> $d/ptxas.txt
grep -A3 "Compiling entry.*path_kernelILi3ELb0" $d/ptxas.txt | tail -2 | tr -s ' ' | sed "s|^|$name: |"
objs=$(ls build/obj/*.o | grep -v mc_engine)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -ccbin /usr/bin/g++ -cudart static \
  -o $d/libcltk_b200.so $objs $d/mc_engine.o -ldl
