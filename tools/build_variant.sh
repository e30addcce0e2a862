#!/bin/bash
# Usage: tools/build_variant.sh NAME "-DFLAG=V ..."  (after the main build)
# Recompiles csrc/dslash.cu with extra flags and links
# paper_1401_3733_b200/liblbcu_NAME.so from it and the main build's other
# objects; select it with LBCU_LIBRARY for A/B timing (tools/tune_hop.py).
set -e
name=$1; flags=$2
root=$(cd "$(dirname "$0")/.." && pwd)
b=$root/build/variant_$name
mkdir -p $b
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
  -I $root/include -I $root/paper_1401_3733_b200/csrc $flags -x cu -c $root/paper_1401_3733_b200/csrc/dslash.cu -o $b/dslash.cu.o
objs=$(ls $root/build/lbcu/*.o | grep -v dslash.cu.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $root/paper_1401_3733_b200/liblbcu_$name.so $b/dslash.cu.o $objs \
  -cudart static -ldl -lpthread -lrt
echo $root/paper_1401_3733_b200/liblbcu_$name.so
