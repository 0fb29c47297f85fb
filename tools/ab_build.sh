#!/bin/bash
# Variant builds of libkcg.so for A/B timing on the GPU box:
#   tools/ab_build.sh NAME "-DKCG_X=0 ..."   ->  tools/_build/libkcg_NAME.so
# (only kcg_count.cu is recompiled; run with KCG_LIB=tools/_build/libkcg_NAME.so)
set -e
cd "$(dirname "$0")/../paper_2002_10047_b200/csrc"
name=$1; shift
mkdir -p ../../tools/_build
/usr/local/cuda/bin/nvcc -std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC \
  --extended-lambda --expt-relaxed-constexpr -I../../include -I. $@ -c kcg_count.cu -o ../../tools/_build/kcg_count_$name.o
objs=$(ls build/*.o | grep -v kcg_count.o)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../tools/_build/libkcg_$name.so $objs ../../tools/_build/kcg_count_$name.o -Xlinker -soname=libkcg.so
rm ../../tools/_build/kcg_count_$name.o
